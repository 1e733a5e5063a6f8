"""Time the K2 prefix match (kvx_match_prefix_batch) on the Config 4 batch,
one instance index of 1M keys, as in bench.py at N=1 (GPU): standalone, and
right after the batch's block hash on the same stream (the hash streams
267 MB of tokens through L2), with and without the index's key table pinned
in L2 (kvx_index_l2_pin).  Every result is checked against the C oracle.
KVX_MATCH_GROUP selects warps per task (1 = warp-per-task kernel)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2407_00079_b200 as pkg  # noqa: E402
from oracle import Oracle  # noqa: E402
from paper_2407_00079_b200.workloads import MatchWorkload  # noqa: E402

mw = MatchWorkload().build()
d = "cuda:0"
s = torch.cuda.Stream(0)
with torch.cuda.stream(s):
    warm_keys, warm_ko = pkg.chain_hash_batch(torch.as_tensor(mw.warm_tokens, device=d),
                                              torch.as_tensor(mw.warm_tok_off, device=d),
                                              mw.block_size, stream=s)
    own = warm_keys[: mw.pool_keys]
    filler = torch.as_tensor(mw.filler_keys(mw.pool_keys - own.numel(), salt=0), device=d)
    content = torch.cat([own, filler])
    idx = pkg.BlockIndex(0, mw.pool_keys)
    idx.insert(content, stream=s)
    tokens = torch.as_tensor(mw.tokens, device=d)
    tok_off = torch.as_tensor(mw.tok_off, device=d)
    keys, key_off = pkg.chain_hash_batch(tokens, tok_off, mw.block_size, stream=s)
s.synchronize()
o = Oracle()
h = o.make_set(content.cpu().numpy())
_, want_len, want_id = o.match_prefix_batch([h], [0], keys.cpu().numpy(), key_off.cpu().numpy())
NREQ = int(os.environ.get("MP_NREQ", mw.n_req))  # the first NREQ requests only (latency probe)
want_len, want_id = want_len[:NREQ], want_id[:NREQ]
bl = torch.empty(NREQ, dtype=torch.int64, device=d)
bi = torch.empty(NREQ, dtype=torch.int32, device=d)
ko_q = key_off[: NREQ + 1]


def match():
    pkg.match_prefix_batch([idx], [0], keys, ko_q, want_lens=False, stream=s, out=(None, bl, bi))


def timed(after_hash, reps=20):
    for _ in range(3):
        if after_hash:
            pkg.chain_hash_batch(tokens, tok_off, mw.block_size, key_off=key_off, keys=keys, stream=s)
        match()
    s.synchronize()
    tot = 0.0
    for _ in range(reps):
        if after_hash:
            pkg.chain_hash_batch(tokens, tok_off, mw.block_size, key_off=key_off, keys=keys, stream=s)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        match()
        e1.record(s)
        s.synchronize()
        tot += e0.elapsed_time(e1)
    ok = np.array_equal(bl.cpu().numpy(), want_len) and np.array_equal(bi.cpu().numpy(), want_id)
    return tot / reps * 1e3, ok


g = os.environ.get("KVX_MATCH_GROUP", "2")
tag = (f"group={g} chains={os.environ.get('KVX_MATCH_CHAINS', '2')} "
       f"order={os.environ.get('KVX_MATCH_ORDER', '0')} occ={os.environ.get('KVX_MATCH_OCC', '0')} "
       f"nreq={NREQ}")
pins = (0, 1) if os.environ.get("MP_PIN", "1") == "1" else (0,)
for pin in pins:
    idx.l2_pin(s, bool(pin))
    for ah in (False, True):
        us, ok = timed(ah)
        print(f"{tag} pin={pin} after_hash={int(ah)} match {us:.1f} us parity={ok}", flush=True)
idx.l2_pin(s, False)
