"""NVLink evidence for the stage-3 paths, one process driving GPUs 0 and 1
(so it can run under ncu, which must never wrap a multi-rank command).

Each mode moves one Config 2 decode wave's worth of one layer range through
the SAME kernels / copies the streamer uses, paged LLaMA2-70B pools (bs 16,
fp16, 32 KiB slabs):
  pull  copy kernel on GPU 1 loading GPU 0's pool (PEER_PULL receiver)
  push  copy kernel on GPU 0 storing into GPU 1's pool (PEER_FUSED sender)
  ce    copy-engine copy of a gathered unit GPU 0 -> GPU 1 (PEER_CE transfer)
and verifies every destination word.  Under ncu the kernels carry the
nvlrx__bytes / nvltx__bytes device counters; for the copy engine (no kernel)
`nvidia-smi nvlink` throughput counters are read around it when available.

  python tests/perf/nvlink_counters.py [--blocks 4096 --layers 4 --reps 5]
"""
import argparse
import json
import os
import subprocess
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2407_00079_b200 import kvx  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--blocks", type=int, default=4096)   # one wave: 16 requests x 256 blocks
ap.add_argument("--layers", type=int, default=4)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--modes", default="pull,push,ce")
args = ap.parse_args()
assert torch.cuda.device_count() >= 2, "needs 2 GPUs"
GB = 1e9
L, bs, n = args.layers, 16, args.blocks
slots = n + 512
kvx.enable_peer(0, 1)
kvx.enable_peer(1, 0)
src = kvx.KVPool(L, bs, 8, 128, 2, slots, 0)
dst = kvx.KVPool(L, bs, 8, 128, 2, slots, 1)
src.fill_synthetic(5)
rng = np.random.default_rng(2)
st = rng.permutation(slots)[:n].astype(np.int32)
dt = rng.permutation(slots)[:n].astype(np.int32)
payload = L * 2 * n * src.slab
st0, dt0 = torch.as_tensor(st, device="cuda:0"), torch.as_tensor(dt, device="cuda:0")
st1, dt1 = torch.as_tensor(st, device="cuda:1"), torch.as_tensor(dt, device="cuda:1")
# views: GPU 0's pool as seen by kernels on GPU 1, GPU 1's pool for GPU 0
src_on1 = kvx.KVPool(L, bs, 8, 128, 2, slots, 1, base_ptr=src.base)
dst_on0 = kvx.KVPool(L, bs, 8, 128, 2, slots, 0, base_ptr=dst.base)
buf0 = kvx.DeviceBuffer(payload, 0)
buf1 = kvx.DeviceBuffer(payload, 1)
eng = kvx.TransferEngine(0)


def nvlink_counters():
    """Per-GPU NVLink data counters from nvidia-smi (KiB), or None."""
    try:
        r = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d"], capture_output=True, text=True,
                           timeout=20)
    except Exception:
        return None
    if r.returncode != 0:
        return None
    out, gpu = {}, None
    for ln in r.stdout.splitlines():
        ln = ln.strip()
        if ln.startswith("GPU "):
            gpu = int(ln.split()[1].rstrip(":"))
            out[gpu] = {"tx_kib": 0, "rx_kib": 0}
        elif gpu is not None and ("Data Tx" in ln or "Data Rx" in ln):
            v = ln.split(":")[-1].strip().split()[0]
            if not v.isdigit():  # "N/A": this driver exposes no throughput counters
                return None
            out[gpu]["tx_kib" if "Data Tx" in ln else "rx_kib"] += int(v)
    return out


def run(mode):
    dst.tensor_view().zero_()
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    dev = 1 if mode == "pull" else 0
    s = torch.cuda.current_stream(dev)
    if mode == "pull":
        fn = lambda: src_on1.copy_to(dst, st1, dt1, 0, L, stream=s)  # noqa: E731
    elif mode == "push":
        fn = lambda: src.copy_to(dst_on0, st0, dt0, 0, L, stream=s)  # noqa: E731
    else:
        src.gather(st0, 0, L, buf0.ptr, stream=torch.cuda.current_stream(0))
        torch.cuda.synchronize(0)
        xs = torch.cuda.ExternalStream(eng.stream_handle, device=0)
        s = xs
        fn = lambda: eng.submit(buf1.ptr, buf0.ptr, payload)  # noqa: E731
    fn()
    torch.cuda.synchronize(dev)
    before = nvlink_counters() if mode == "ce" else None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(args.reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize(dev)
    after = nvlink_counters() if mode == "ce" else None
    ms = e0.elapsed_time(e1) / args.reps
    # parity: every destination word
    if mode == "ce":
        dst.scatter(dt1, 0, L, buf1.ptr, stream=torch.cuda.current_stream(1))
    bad = torch.zeros(1, dtype=torch.int64, device="cuda:1")
    dst.verify(dt1, 5, st1, 0, L, counter=bad)
    torch.cuda.synchronize(1)
    rec = {"mode": mode, "payload_bytes": payload, "ms": ms, "gbs": payload / (ms / 1e3) / GB,
           "mismatched_words": int(bad.item())}
    if before and after:
        rec["nvidia_smi_nvlink_kib"] = {
            g: {k: after[g][k] - before[g][k] for k in ("tx_kib", "rx_kib")} for g in after}
        rec["nvidia_smi_note"] = f"counter deltas over the {args.reps + 0} timed copies"
    return rec


res = [run(m) for m in args.modes.split(",")]
for r in res:
    print(json.dumps(r), flush=True)
assert all(r["mismatched_words"] == 0 for r in res)
