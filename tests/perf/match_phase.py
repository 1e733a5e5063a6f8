"""Time the K2 prefix match (kvx_match_prefix_batch) on the Config 4 batch,
one instance index of 1M keys, as in bench.py at N=1 (GPU)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2407_00079_b200 as pkg  # noqa: E402
from paper_2407_00079_b200.workloads import MatchWorkload  # noqa: E402

mw = MatchWorkload().build()
d = "cuda:0"
warm_keys, warm_ko = pkg.chain_hash_batch(torch.as_tensor(mw.warm_tokens, device=d),
                                          torch.as_tensor(mw.warm_tok_off, device=d), mw.block_size)
own = warm_keys[: mw.pool_keys]
filler = torch.as_tensor(mw.filler_keys(mw.pool_keys - own.numel(), salt=0), device=d)
idx = pkg.BlockIndex(0, mw.pool_keys)
idx.insert(torch.cat([own, filler]))
tok_off = torch.as_tensor(mw.tok_off, device=d)
keys, key_off = pkg.chain_hash_batch(torch.as_tensor(mw.tokens, device=d), tok_off, mw.block_size)
for _ in range(3):
    _, bl, bi = pkg.match_prefix_batch([idx], [0], keys, key_off, want_lens=False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    pkg.match_prefix_batch([idx], [0], keys, key_off, want_lens=False, out=(None, bl, bi))
e1.record()
torch.cuda.synchronize()
lens = bl.cpu().numpy()
n = np.diff(key_off.cpu().numpy())
print(f"match: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us  probes={int(np.minimum(lens + 1, n).sum())} "
      f"max_len={int(lens.max())} mean_len={lens.mean():.0f} checksum={int(lens.sum())}")
