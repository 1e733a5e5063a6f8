"""Time kvx_chain_hash_batch on the Config 4 batch (GPU).  With
KVX_HASH_FOLD_SMS=-1 the kernel only produces content hashes (keys are then
NOT final) -- used to split the stage-1a time into production and fold."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2407_00079_b200 as pkg  # noqa: E402
from paper_2407_00079_b200.workloads import MatchWorkload  # noqa: E402

mw = MatchWorkload().build()
tok_np, off_np = mw.tokens, mw.tok_off
shard = os.environ.get("HASH_SHARD")  # "k/N": rank k's token-balanced shard of the batch
if shard:
    from bench import shard_by_tokens  # noqa: E402
    k, n = (int(x) for x in shard.split("/"))
    r0, r1 = shard_by_tokens(off_np, n)[k]
    tok_np = tok_np[off_np[r0]:off_np[r1]]
    off_np = off_np[r0:r1 + 1] - off_np[r0]
tokens = torch.as_tensor(tok_np, device="cuda")
tok_off = torch.as_tensor(off_np, device="cuda")
key_off = pkg.kvx.key_offsets(tok_off, 16)
keys = torch.empty(int(key_off[-1].item()), dtype=torch.int64, device="cuda")
for _ in range(3):
    pkg.chain_hash_batch(tokens, tok_off, 16, key_off=key_off, keys=keys)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    pkg.chain_hash_batch(tokens, tok_off, 16, key_off=key_off, keys=keys)
e1.record()
torch.cuda.synchronize()
ok = "n/a"
if os.environ.get("KVX_HASH_FOLD_SMS") != "-1":  # keys are final: check them all
    from oracle import Oracle
    want, _ = Oracle().block_hash_batch(tok_np, off_np, 16)
    ok = bool((keys.cpu().numpy() == want).all())
print(f"shard={shard or 'all'} kernel={os.environ.get('KVX_HASH_KERNEL', 'halfwarp')} "
      f"fold_sms={os.environ.get('KVX_HASH_FOLD_SMS', 'auto')} "
      f"prio={os.environ.get('KVX_HASH_PRIO', '1')} warps={os.environ.get('KVX_HASH_HW_WARPS', '12')} "
      f"hash batch: {e0.elapsed_time(e1) / 10 * 1e3:.1f} us parity={ok}")
