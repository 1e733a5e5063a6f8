"""Does a PEER_PULL receiver starve the decode GPU while it waits for a slow
prefill?  Two processes (torchrun, one per GPU).  The sender publishes one
layer of a 2,048-token chunk (128 blocks x 2 x 32 KiB = 8 MiB) every
`--delay-us` (a sleep kernel on its queue stands in for the prefill of that
layer); the receiver enqueues all 80 units in one recv call (the units are
chained by programmatic dependent launch) and, on another stream, runs a
bf16 GEMM loop standing in for decode work.  Reported per run: the GEMM's
TFLOP/s while the transfer is in flight vs alone, and the transfer time.

  torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tests/perf/pull_starvation.py
  (KVX_PULL_GATE=gate|inline|stream selects how the receiver waits)
"""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2407_00079_b200 as pkg  # noqa: E402
from paper_2407_00079_b200.cluster import exchange_with_peer, pair_topology  # noqa: E402
from paper_2407_00079_b200.streamer import Streamer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--delay-us", type=float, default=200.0)
ap.add_argument("--layers", type=int, default=80)
args = ap.parse_args()
rank = int(os.environ["RANK"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device(f"cuda:{rank}"))
role = pair_topology(2, rank)
L, bs, n = args.layers, 16, 128
slots = 256
d = f"cuda:{rank}"
pool = pkg.KVPool(L, bs, 8, 128, 2, slots, rank)
if role.role == "prefill":
    pool.fill_synthetic(3)
    st = Streamer("peer_pull", "sender", pool, None)
else:
    pool.tensor_view().zero_()
    st = Streamer("peer_pull", "receiver", None, pool)
peer = exchange_with_peer(role, {"blob": st.export()})
desc = dict(layers=L, block_size=bs, heads=8, head_dim=128, dtype_bytes=2, slots=slots)
st.connect(peer["blob"], desc)
rng = np.random.default_rng(0)
src_t = torch.as_tensor(rng.permutation(slots)[:n].astype(np.int32), device=d)
dst_t = torch.as_tensor(rng.permutation(slots)[:n].astype(np.int32), device=d)
cycles = int(args.delay_us * 1e-6 * 1.9e9)


A = B = C_ = None


def gemm_rate(stream, iters=20):
    """`iters` back-to-back bf16 8192^3 GEMMs on `stream`; TFLOP/s by CUDA
    events around the whole loop (enqueued at once: they run as soon as the
    SMs let them)."""
    global A, B, C_
    if A is None:
        A = torch.randn(8192, 8192, dtype=torch.bfloat16, device=d)
        B = torch.randn(8192, 8192, dtype=torch.bfloat16, device=d)
        C_ = torch.empty(8192, 8192, dtype=torch.bfloat16, device=d)
        torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(iters):
            torch.matmul(A, B, out=C_)
        e1.record(stream)
    return e0, e1, iters


def rate(ev):
    e0, e1, k = ev
    return 2 * 8192 ** 3 * k / (e0.elapsed_time(e1) / 1e3) / 1e12


def one_step(with_gemm):
    dist.barrier()
    torch.cuda.synchronize()
    s = torch.cuda.ExternalStream(st.stream.cuda_stream, device=rank)
    res = {}
    if role.role == "prefill":
        for layer in range(L):  # one layer's KV "produced" every delay_us
            with torch.cuda.stream(s):
                torch.cuda._sleep(cycles)
            st.send(src_t, None, layer, layer + 1, 0, 1)
        st.finish(torch.cuda.current_stream())
        torch.cuda.synchronize()
    else:
        gs = torch.cuda.Stream(rank)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        st.recv(dst_t, 0, L, 0, 1, src_table=src_t)
        e1.record(s)
        st.finish(torch.cuda.current_stream())
        g = gemm_rate(gs) if with_gemm else None  # ~14 ms of GEMMs inside the ~16 ms transfer
        torch.cuda.synchronize()
        if g is not None:
            res["gemm_tflops_during_transfer"] = rate(g)
            res["gemm_window_ms"] = g[0].elapsed_time(g[1])
            res["gemm_started_after_transfer_start_ms"] = e0.elapsed_time(g[0])
        st.check()
        res["transfer_ms"] = e0.elapsed_time(e1)
        bad = torch.zeros(1, dtype=torch.int64, device=d)
        pool.verify(dst_t, 3, src_t, 0, L, counter=bad)
        torch.cuda.synchronize()
        res["mismatched_words"] = int(bad.item())
    dist.barrier()
    return res


one_step(False)
alone = None
if role.role == "decode":
    ev = gemm_rate(torch.cuda.Stream(rank))
    torch.cuda.synchronize()
    alone = rate(ev)
dist.barrier()
r = one_step(True)
if role.role == "decode":
    print(json.dumps({"mode": os.environ.get("KVX_PULL_GATE", "gate"), "delay_us": args.delay_us,
                      "gemm_alone_tflops": alone, **r}), flush=True)
dist.barrier()
dist.destroy_process_group()
