"""Critical-path probe of the block-hash kernel: batches of N equal requests
of T tokens (bs 16), N = 1 (one half-warp: the bare per-step latency of the
key chain), one per SM, one per SM sub-partition, ... up to the Config 4
request count.  Prints us per batch and cycles per 16-token step at the
measured SM clock.  python tests/perf/hash_latency.py"""
import os
import subprocess
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2407_00079_b200 as pkg  # noqa: E402
from oracle import Oracle  # noqa: E402

T = int(os.environ.get("HL_TOKENS", "24576"))
o = Oracle()
rng = np.random.default_rng(0)
NS = [int(x) for x in os.environ.get("HL_NS", "1,2,32,148,296,592,1184,1776,2368,3552,4096").split(",")]
for n in NS:
    lens = np.full(n, T, dtype=np.int64)
    tok_off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    tokens = rng.integers(0, 32000, size=int(tok_off[-1])).astype(np.int32)
    t, to = torch.as_tensor(tokens, device="cuda"), torch.as_tensor(tok_off, device="cuda")
    ko = pkg.kvx.key_offsets(to, 16)
    keys = torch.empty(int(ko[-1].item()), dtype=torch.int64, device="cuda")
    for _ in range(3):
        pkg.chain_hash_batch(t, to, 16, key_off=ko, keys=keys)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        pkg.chain_hash_batch(t, to, 16, key_off=ko, keys=keys)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 5 * 1e3
    if n <= 32:
        want, _ = o.block_hash_batch(tokens, tok_off, 16)
        assert (keys.cpu().numpy() == want).all()
    steps = -(-(T // 16) // 15) * 16
    clk = float(subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits",
                                "-i", "0"], capture_output=True, text=True).stdout.split()[0] or 0)
    print(f"n={n} T={T} batch {us:.1f} us  {us * 1e-6 * clk * 1e6 / steps:.0f} cycles/step "
          f"(clock now {clk:.0f} MHz)", flush=True)
