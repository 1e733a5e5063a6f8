"""torchrun worker for tests/test_gpu_xmatch.py: each rank holds ONE prefill
instance's block index; kvx_xmatch_run (match kernel with NVLink remote
atomics + stream flags, no collective) must equal find_best_prefix_match over
all instances queried on one GPU, over several batches of different sizes
(exercises the double-buffered, re-zeroed result buffers)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_00079_b200 as pkg  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
# KVX_SHARE_GPU=1: every rank on cuda:0 (processes sharing one GPU; gloo
# handshake) -- the remote atomics and flags then target the same device
share = os.environ.get("KVX_SHARE_GPU") == "1"
dev = 0 if share else rank
torch.cuda.set_device(dev)
if share:
    dist.init_process_group("gloo")
else:
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{dev}"))
d = f"cuda:{dev}"
rng = np.random.default_rng(5)  # same inputs on every rank
n_req = 96
lens = rng.integers(0, 160, n_req)
off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
keys = rng.integers(1, 1 << 62, int(off[-1]), dtype=np.int64)
# instance j holds a random-length prefix of every request's chain; equal
# lengths across instances are frequent (tie-break: lowest instance id wins)
held = rng.integers(0, 5, (world, n_req)) * (lens // 4 + 1)
ids = [world - j + 3 for j in range(world)]  # higher rank -> lower id


def instance_keys(j):
    parts = [keys[off[r]: off[r] + min(int(held[j, r]), int(lens[r]))] for r in range(n_req)]
    return torch.as_tensor(np.concatenate(parts) if parts else keys[:0], device=d)


def index_of(j):
    ix = pkg.BlockIndex(dev, 4096)
    ix.insert(instance_keys(j))
    return ix


mine = index_of(rank)
everyone = [index_of(j) for j in range(world)]
xm = pkg.kvx.XMatch(dev, rank, world, max_req=n_req)
blobs = [None] * world
dist.all_gather_object(blobs, xm.export())
for b in blobs:
    xm.connect(b)
dk = torch.as_tensor(keys, device=d)
for step, n in enumerate([n_req, 37, n_req, 1, 64, n_req]):
    ko = torch.as_tensor(off[: n + 1], device=d)
    s = torch.cuda.current_stream()
    best_len, best_id = xm.run([mine], [ids[rank]], dk, ko, stream=s)
    _, ref_len, ref_id = pkg.match_prefix_batch(everyone, ids, dk, ko, want_lens=False, stream=s)
    torch.cuda.synchronize()
    assert torch.equal(best_len, ref_len), (step, best_len, ref_len)
    assert torch.equal(best_id, ref_id), (step, best_id, ref_id)
dist.barrier()
del xm
torch.cuda.synchronize()
dist.destroy_process_group()
if rank == 0:
    print("XMATCH OK")
