"""CPU, world_size 2 and 4 over gloo: prefill/decode pairing, the pair
handshake and the max-over-ranks timing reduction used by bench.py --gpus N."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2407_00079_b200.cluster import (exchange_with_peer, max_over_ranks, pair_topology,
                                           sum_over_ranks)


def test_pair_topology():
    assert pair_topology(1, 0).role == "local"
    roles = [pair_topology(8, r) for r in range(8)]
    assert [r.role for r in roles] == ["prefill"] * 4 + ["decode"] * 4
    assert [r.peer for r in roles] == [4, 5, 6, 7, 0, 1, 2, 3]
    assert [r.pair for r in roles] == [0, 1, 2, 3, 0, 1, 2, 3]
    assert all(r.pairs == 4 for r in roles)
    with pytest.raises(ValueError):
        pair_topology(3, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    role = pair_topology(world, rank)
    # decode sends its (fake) IPC handles + block tables, prefill its flag handle
    payload = {"rank": rank, "role": role.role,
               "pool": bytes([rank]) * 64 if role.role == "decode" else None,
               "tables": [rank * 100 + i for i in range(3)]}
    peer = exchange_with_peer(role, payload)
    slowest = max_over_ranks(1.0 + rank)
    total = sum_over_ranks(2.0)
    q.put((rank, role.role, peer["rank"], peer["role"], peer["pool"], peer["tables"], slowest,
           total))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_handshake_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    half = world // 2
    for rank, role, peer_rank, peer_role, peer_pool, peer_tables, slowest, total in res:
        assert slowest == float(world) and total == 2.0 * world
        if rank < half:
            assert role == "prefill" and peer_rank == rank + half and peer_role == "decode"
            assert peer_pool == bytes([rank + half]) * 64
        else:
            assert role == "decode" and peer_rank == rank - half and peer_pool is None
        assert peer_tables == [peer_rank * 100 + i for i in range(3)]
