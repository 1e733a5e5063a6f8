"""Phase profile of the K1d hash kernel (KVX_HASH_KERNEL=fold, GPU): cycles
each producer / folding warp spends per phase, from clock64 stamps inside the
kernel (KVX_HASH_PROFILE=1; measurement only).  Workload: the Config 4 batch,
or HP_EQUAL=n equal requests of 24,576 tokens."""
import ctypes as C
import os
import sys

os.environ["KVX_HASH_KERNEL"] = "fold"
os.environ["KVX_HASH_PROFILE"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2407_00079_b200 as pkg  # noqa: E402
from paper_2407_00079_b200 import kvx  # noqa: E402
from paper_2407_00079_b200.workloads import MatchWorkload  # noqa: E402

n_eq = int(os.environ.get("HP_EQUAL", "0"))
if n_eq:
    tok_np = np.random.default_rng(1).integers(0, 32000, n_eq * 24576).astype(np.int32)
    off_np = np.arange(n_eq + 1, dtype=np.int64) * 24576
else:
    mw = MatchWorkload().build()
    tok_np, off_np = mw.tokens, mw.tok_off
tokens = torch.as_tensor(tok_np, device="cuda")
tok_off = torch.as_tensor(off_np, device="cuda")
key_off = pkg.kvx.key_offsets(tok_off, 16)
keys = torch.empty(int(key_off[-1].item()), dtype=torch.int64, device="cuda")
for _ in range(3):
    pkg.chain_hash_batch(tokens, tok_off, 16, key_off=key_off, keys=keys)
f = kvx._L.kvx_hash_profile
f.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
buf = (C.c_ulonglong * 8016)()
f(buf, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
runs = 10
for _ in range(runs):
    pkg.chain_hash_batch(tokens, tok_off, 16, key_off=key_off, keys=keys)
e1.record()
torch.cuda.synchronize()
f(buf, 0)
v = [int(x) for x in buf[:14]]
if os.environ.get("HP_TRACE"):  # one more launch, traced on SM 0
    f(buf, 1)
    pkg.chain_hash_batch(tokens, tok_off, 16, key_off=key_off, keys=keys)
    torch.cuda.synchronize()
    f(buf, 0)
    arr = np.frombuffer(buf, dtype=np.uint64).copy()
    n_ev = min(int(arr[8]), 4000)
    ev = arr[16:16 + 2 * n_ev].reshape(-1, 2)
    out = os.environ["HP_TRACE"]
    np.save(out, ev)
    print(f"trace: {n_ev} events -> {out}")
W = int(os.environ.get("KVX_HASH_FOLD_CTA_WARPS", "28"))
share = int(os.environ.get("KVX_HASH_FOLD_SHARE", "1"))
P = sum(1 for w in range(W - 2) if w % 4 != (W - 1) % 4 or w // 4 < share)
sms = torch.cuda.get_device_properties(0).multi_processor_count
us = e0.elapsed_time(e1) / runs * 1e3
prod = v[0:5]
tot = sum(prod)
names = ["claim", "issue", "wait", "hash", "publish"]
print(f"warps={W} share={share} producers={P} n_eq={n_eq} batch {us:.1f} us (with clock64 stamps)")
print("producer cycles per warp per launch: " + ", ".join(
    f"{n} {x / runs / (sms * P):.0f} ({x / tot:.1%})" for n, x in zip(names, prod)))
fold = v[5] + v[6]
print(f"folder cycles per launch: idle {v[5] / runs / sms:.0f} ({v[5] / max(fold, 1):.1%}), "
      f"windows {v[6] / runs / sms:.0f}; iterations per SM {v[7] / runs / sms:.1f}")
print(f"dispatcher per SM per launch: full-ring stalls {v[10] / runs / sms:.0f}, "
      f"tasks {v[11] / runs / sms:.0f}; idle {v[12] / runs / sms:.0f} cycles, "
      f"filling {v[13] / runs / sms:.0f} cycles")
