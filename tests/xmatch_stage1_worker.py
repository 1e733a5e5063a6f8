"""torchrun worker for tests/test_gpu_xmatch.py: request-sharded stage 1 with
the key exchange inside the match kernel (kvx_xmatch_hash_match).  Each rank
hashes its shard of the batch into its own key buffer, and each rank's match
kernel follows the whole batch (peer shards through NVLink loads) against
the rank's ONE prefill instance.  Must equal chain_hash_batch over the whole batch
and find_best_prefix_match over all instances on one GPU, over several steps
and two batch shapes (exercises both key-buffer halves and the flags).
KVX_SHARE_GPU=1 (ranks sharing cuda:0): the call must refuse (KVX_EINVAL)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_00079_b200 as pkg  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
share = os.environ.get("KVX_SHARE_GPU") == "1"
dev = 0 if share else rank
torch.cuda.set_device(dev)
if share:
    dist.init_process_group("gloo")
else:
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{dev}"))
d = f"cuda:{dev}"
rng = np.random.default_rng(11)  # same inputs on every rank


def batch(n_req, max_tok, misalign):
    lens = rng.integers(0, max_tok, n_req)
    if n_req > 3:
        lens[3] = 0
    off = (np.concatenate([[0], np.cumsum(lens)]) + misalign).astype(np.int64)
    toks = rng.integers(0, 32000, int(off[-1]) + 8).astype(np.int32)
    return torch.as_tensor(toks, device=d), torch.as_tensor(off, device=d), off


# a large batch, a small one, and one whose single request leaves every
# other rank's shard empty
# (and one at block size 32)
batches = [batch(300, 6000, 3) + (16,), batch(180, 2000, 0) + (16,), batch(1, 9000, 1) + (16,),
           batch(120, 8000, 2) + (32,)]
ids = [world - j + 5 for j in range(world)]
plans = []
max_keys = 0
for toks, toff, off_np, bs in batches:
    keys_ref, koff = pkg.chain_hash_batch(toks, toff, bs)
    n_req = len(off_np) - 1
    koff_np = koff.cpu().numpy()
    lens = np.diff(koff_np)
    held = rng.integers(0, 5, (world, n_req)) * (lens // 4 + 1)
    kr = keys_ref.cpu().numpy()

    def index_of(j, kr=kr, koff_np=koff_np, held=held, lens=lens):
        parts = [kr[koff_np[r]: koff_np[r] + min(int(held[j, r]), int(lens[r]))]
                 for r in range(n_req)]
        ix = pkg.BlockIndex(dev, 1 << 16)
        ix.insert(torch.as_tensor(np.concatenate(parts), device=d))
        return ix

    everyone = [index_of(j) for j in range(world)]
    _, ref_len, ref_id = pkg.match_prefix_batch(everyone, ids, keys_ref, koff, want_lens=False)
    bounds = [j * n_req // world for j in range(world)] + [n_req]
    plans.append((toks, toff, koff, keys_ref, ref_len, ref_id, everyone[rank], bounds, bs))
    max_keys = max(max_keys, int(koff_np[-1]))

xm = pkg.kvx.XMatch(dev, rank, world, max_req=400)
xm.key_buffer(max_keys)
blobs = [None] * world
dist.all_gather_object(blobs, xm.export())
for b in blobs:
    xm.connect(b)
torch.cuda.synchronize()
s = torch.cuda.current_stream()
if share:
    toks, toff, koff, *_rest, mine, bounds, bs = plans[0]
    try:
        xm.hash_match(toks, toff, bounds, bs, koff, [mine], [ids[rank]], stream=s)
        raise SystemExit("shared GPU: kvx_xmatch_hash_match did not refuse")
    except pkg.kvx.ValidationError:
        pass
else:
    for step, which in enumerate([0, 0, 1, 0, 2, 1, 3, 1, 0, 2, 3]):
        toks, toff, koff, keys_ref, ref_len, ref_id, mine, bounds, bs = plans[which]
        best_len, best_id, keys = xm.hash_match(toks, toff, bounds, bs, koff, [mine],
                                                [ids[rank]], stream=s)
        torch.cuda.synchronize()
        pkg.kvx.check(pkg.kvx._L.kvx_hash_match_check(None))
        k0, k1 = int(koff[bounds[rank]].item()), int(koff[bounds[rank + 1]].item())
        assert torch.equal(keys[k0:k1], keys_ref[k0:k1]), ("keys", step)
        assert torch.equal(best_len, ref_len), ("best_len", step)
        assert torch.equal(best_id, ref_id), ("best_id", step)
dist.barrier()
del xm
torch.cuda.synchronize()
dist.destroy_process_group()
if rank == 0:
    print("XMATCH STAGE1 OK")
