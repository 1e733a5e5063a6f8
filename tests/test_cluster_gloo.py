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


def test_shard_by_tokens_covers_batch():
    """Stage-1 request sharding (bench.py --gpus N, "sharded" object): the
    shards are contiguous, disjoint, cover every request once, and balance
    tokens to within one request per boundary."""
    import numpy as np

    from bench import shard_by_tokens
    rng = np.random.default_rng(3)
    for world in (1, 2, 3, 4, 8):
        for n in (0, 1, 5, 4096):
            lens = rng.integers(0, 24577, size=n)
            tok_off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
            sh = shard_by_tokens(tok_off, world)
            assert len(sh) == world and sh[0][0] == 0 and sh[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(sh, sh[1:]))
            assert all(r0 <= r1 for r0, r1 in sh)
            if n > 100:
                tot = [int(tok_off[r1] - tok_off[r0]) for r0, r1 in sh]
                assert max(tot) - min(tot) <= 2 * int(lens.max())


def _shard_worker(rank, world, port, q):
    """Every rank takes its shard; the all-gathered shards rebuild the batch."""
    import numpy as np

    from bench import shard_by_tokens
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(11)  # same batch on every rank
    lens = rng.integers(1, 3000, size=257)
    tok_off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    r0, r1 = shard_by_tokens(tok_off, world)[rank]
    key_off = np.concatenate([[0], np.cumsum((lens + 15) // 16)])
    mine = list(range(int(key_off[r0]), int(key_off[r1])))  # key positions this rank hashes
    out = [None] * world
    dist.all_gather_object(out, mine)
    q.put((rank, sorted(k for part in out for k in part) == list(range(int(key_off[-1])))))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_keys_cover_batch_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res)
