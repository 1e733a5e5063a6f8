"""Request-sharded stage 1 over the GPUs of one box (torchrun, one rank per
GPU): the hash of one shard alone, the separate step (hash shard ->
kvx_xmatch_share_keys -> kvx_xmatch_run) and kvx_xmatch_hash_match (no
parity check here -- the bench and tests/test_gpu_xmatch.py check it)."""
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2407_00079_b200 as pkg  # noqa: E402
from bench import Stage1Batch, shard_by_tokens  # noqa: E402
from paper_2407_00079_b200.workloads import MatchWorkload  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device(f"cuda:{rank}"))
d = f"cuda:{rank}"
s = torch.cuda.Stream(rank)
mw = MatchWorkload(seed=4).build()
B = Stage1Batch(mw, rank, s)
idx = B.index(rank, world)
xm = pkg.kvx.XMatch(rank, rank, world, mw.n_req)
keys = xm.key_buffer(B.n_blocks)
blobs = [None] * world
dist.all_gather_object(blobs, xm.export())
for b in blobs:
    xm.connect(b)
r0, r1 = shard_by_tokens(mw.tok_off, world)[rank]
k0, k1 = int(B.key_off_host[r0]), int(B.key_off_host[r1])
with torch.cuda.stream(s):
    bl = torch.empty(mw.n_req, dtype=torch.int64, device=d)
    bi = torch.empty(mw.n_req, dtype=torch.int32, device=d)


def sep():
    pkg.chain_hash_batch(B.tokens, B.tok_off[r0:r1 + 1], mw.block_size,
                         key_off=B.key_off[r0:r1 + 1], keys=keys, stream=s)
    xm.share_keys(k0, k1, stream=s)
    xm.run([idx], [rank], keys, B.key_off, out=(bl, bi), stream=s)


def hash_only():
    pkg.chain_hash_batch(B.tokens, B.tok_off[r0:r1 + 1], mw.block_size,
                         key_off=B.key_off[r0:r1 + 1], keys=keys, stream=s)


bounds = [0] + [b for _, b in shard_by_tokens(mw.tok_off, world)]


def fused():
    xm.hash_match(B.tokens, B.tok_off, bounds, mw.block_size, B.key_off, [idx], [rank],
                  out=(bl, bi), stream=s)


def timeit(fn, n=10):
    for _ in range(3):
        fn()
    s.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(n):
        fn()
    e1.record(s)
    s.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / n * 1e3], device=d)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


res = {}
if os.environ.get("XS1_ONLY") != "fused":
    res["hash_shard"] = timeit(hash_only)
    res["separate"] = timeit(sep)
res["fused"] = timeit(fused)
if rank == 0:
    print(f"world={world}: " + ", ".join(f"{k} {v:.1f} us" for k, v in res.items()))
del xm
dist.destroy_process_group()
