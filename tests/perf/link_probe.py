"""NVLink probe between rank 0 (sender) and rank 1 (receiver), 2 processes:
copy-engine copies on 1, 2 and 4 queues at once, and SM copy kernels pushing
(rank 0 stores into rank 1's memory) or pulling (rank 1 loads from rank 0).
torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tests/perf/link_probe.py"""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2407_00079_b200 import kvx  # noqa: E402

rank = int(os.environ["RANK"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device(f"cuda:{rank}"))
NB = 4 << 30
mine = kvx.DeviceBuffer(NB, rank)
handles = [None, None]
dist.all_gather_object(handles, kvx.ipc_export(mine.ptr))
peer = kvx.ipc_open(handles[1 - rank], rank)
GB = 1e9


def timed(fn, reps=3):
    """Local timing only -- callers keep the collective calls symmetric."""
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s = torch.cuda.current_stream()
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


res = {}
if rank == 0:
    for q in (1, 2, 4):
        engs = [kvx.TransferEngine(0) for _ in range(q)]

        def ce():
            part = NB // q
            cur = torch.cuda.current_stream()
            ts = [e.submit(peer + i * part, mine.ptr + i * part, part, after_stream=cur)
                  for i, e in enumerate(engs)]
            for e, t in zip(engs, ts):
                e.wait_stream(t, cur)
        res[f"ce_{q}q"] = NB / (timed(ce) / 1e3) / GB
# SM copy kernels over a flat "pool" (1 layer, slab = 1 MiB, identity tables)
SLAB = 1 << 20
n = NB // (2 * SLAB)
desc = dict(layers=1, block_size=512, heads=8, head_dim=128, dtype_bytes=2, slots=n)
local = kvx.KVPool(**desc, device=rank, base_ptr=mine.ptr)
remote = kvx.KVPool(**desc, device=rank, base_ptr=peer)
tab = torch.arange(n, dtype=torch.int32, device=f"cuda:{rank}")
if rank == 0:
    res["sm_push"] = NB / (timed(lambda: local.copy_to(remote, tab, tab, 0, 1)) / 1e3) / GB
dist.barrier()
if rank == 1:
    res["sm_pull"] = NB / (timed(lambda: remote.copy_to(local, tab, tab, 0, 1)) / 1e3) / GB
out = [None, None]
dist.all_gather_object(out, res)
if rank == 0:
    merged = {**out[0], **out[1]}
    print({k: round(v, 1) for k, v in merged.items()})
dist.barrier()
dist.destroy_process_group()
