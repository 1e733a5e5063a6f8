"""GPU parity: K1 block hash and K2 prefix match (through the C ABI) against
the reference's golden vectors (tests/golden, from oracle/_ref) and the C
restatement (oracle/) on seeded inputs.  Bit-exact integer equality."""
import numpy as np
import pytest
import torch

from conftest import golden

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


def _t(a, dtype):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device=DEV)


@pytest.mark.parametrize("bs", [1, 5, 16, 64])
def test_block_hash_golden(kvx, bs):
    g = golden("block_hash.npz")
    keys, ko = kvx.chain_hash_batch(_t(g[f"bs{bs}_tokens"], torch.int32),
                                    _t(g[f"bs{bs}_tok_off"], torch.int64), bs)
    assert np.array_equal(keys.cpu().numpy(), g[f"bs{bs}_keys"])


@pytest.mark.parametrize("bs,misalign", [(16, 0), (16, 3), (32, 0), (7, 1), (512, 0)])
def test_block_hash_random_vs_oracle(kvx, oracle_lib, bs, misalign):
    rng = np.random.default_rng(bs * 10 + misalign)
    lens = rng.integers(0, 40 * bs, size=97)
    lens[5] = 0
    lens[6] = 1
    tok_off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64) + misalign
    tokens = rng.integers(0, 32000, size=int(tok_off[-1]) + 8).astype(np.int32)
    want, wko = oracle_lib.block_hash_batch(tokens, tok_off, bs)
    keys, ko = kvx.chain_hash_batch(_t(tokens, torch.int32), _t(tok_off, torch.int64), bs)
    assert np.array_equal(ko.cpu().numpy(), wko)
    assert np.array_equal(keys.cpu().numpy(), want)


def test_block_hash_many_small_requests(kvx, oracle_lib):
    """More requests than folding lanes (each lane folds several requests) and
    many empty / sub-block requests."""
    rng = np.random.default_rng(77)
    lens = rng.integers(0, 60, size=40000)
    tok_off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    tokens = rng.integers(0, 32000, size=int(tok_off[-1])).astype(np.int32)
    want, _ = oracle_lib.block_hash_batch(tokens, tok_off, 16)
    keys, _ = kvx.chain_hash_batch(_t(tokens, torch.int32), _t(tok_off, torch.int64), 16)
    assert np.array_equal(keys.cpu().numpy(), want)


def test_scalar_chain_hash(kvx):
    g = golden("chain_hash.npz")
    for p, c, o in zip(g["prev"][:64], g["content"][:64], g["out"][:64]):
        assert kvx.chain_hash(int(p), int(c)) == int(o)


def _index(kvx, keys):
    idx = kvx.BlockIndex(0, max(len(keys), 16))
    if len(keys):
        idx.insert(_t(keys, torch.int64))
    return idx


def test_match_prefix_reference_kats(kvx):
    # proj/tests/test_kvcache.cpp:37-73 and proj/tests/test_conductor.cpp:81-113
    chain = _t([1, 2, 3], torch.int64)
    off = _t([0, 3], torch.int64)
    for content, want in [([], 0), ([1], 1), ([3], 0), ([1, 2, 3], 3)]:
        lens, bl, bi = kvx.match_prefix_batch([_index(kvx, content)], [0], chain, off)
        assert lens.item() == want and bl.item() == want and bi.item() == 0
    chain = _t(np.arange(8), torch.int64)
    off = _t([0, 8], torch.int64)
    cases = [([[], []], (0, 0)), ([range(3), range(7), range(7)], (7, 1)),
             ([range(2), range(8)], (8, 1))]
    for contents, want in cases:
        idx = [_index(kvx, list(c)) for c in contents]
        _, bl, bi = kvx.match_prefix_batch(idx, list(range(len(idx))), chain, off)
        assert (bl.item(), bi.item()) == want
    with pytest.raises(kvx.ValidationError):
        kvx.match_prefix_batch([], [], chain, off)


def test_match_states_golden(kvx):
    """400 randomized states (criterion-4 shape) -- expected values come from
    kvref::CachePool::match_prefix and kvref::find_best_prefix_match."""
    g = golden("match_states.npz")
    ii = 0
    for s in range(len(g["inst_cnt"])):
        n_inst = int(g["inst_cnt"][s])
        idx, ids = [], []
        for _ in range(n_inst):
            lo, hi = g["inst_off"][ii], g["inst_off"][ii + 1]
            idx.append(_index(kvx, g["inst_keys"][lo:hi]))
            ids.append(int(g["inst_ids"][ii]))
            ii += 1
        q = g["q_keys"][g["q_off"][s]:g["q_off"][s + 1]]
        lens, bl, bi = kvx.match_prefix_batch(idx, ids, _t(q, torch.int64),
                                              _t([0, len(q)], torch.int64))
        assert lens[0].cpu().tolist() == g["lens"][ii - n_inst:ii].tolist(), s
        assert (bl.item(), bi.item()) == (int(g["best_len"][s]), int(g["best_id"][s])), s


def _forest(rng, n_req, n_sessions, min_len, max_len):
    """Session-forest requests: each request extends a random prefix of its
    session's chain (oracles.hpp:285-308 structure)."""
    chains = [rng.integers(0, 1 << 62, size=max_len, dtype=np.int64) for _ in range(n_sessions)]
    reqs = []
    for _ in range(n_req):
        c = chains[int(rng.integers(0, n_sessions))]
        n = int(rng.integers(min_len, max_len + 1))
        share = int(rng.integers(0, n + 1))
        fresh = rng.integers(0, 1 << 62, size=n - share, dtype=np.int64)
        reqs.append(np.concatenate([c[:share], fresh]))
    return reqs


@pytest.mark.parametrize("n_inst", [1, 3, 8, 64])
def test_match_batch_random_vs_oracle(kvx, oracle_lib, n_inst):
    rng = np.random.default_rng(1000 + n_inst)
    reqs = _forest(rng, 300, 12, 0, 400)
    key_off = np.concatenate([[0], np.cumsum([len(r) for r in reqs])]).astype(np.int64)
    keys = np.concatenate(reqs).astype(np.int64)
    contents = []
    for i in range(n_inst):
        pick = rng.choice(len(reqs), size=20, replace=False)
        ks = [reqs[p][: int(rng.integers(0, len(reqs[p]) + 1))] for p in pick]
        ks.append(rng.integers(0, 1 << 62, size=50, dtype=np.int64))
        contents.append(np.concatenate(ks).astype(np.int64))
    ids = rng.permutation(n_inst).astype(np.int32) - 3
    idx = [_index(kvx, c) for c in contents]
    lens, bl, bi = kvx.match_prefix_batch(idx, ids.tolist(), _t(keys, torch.int64),
                                          _t(key_off, torch.int64))
    sets = [oracle_lib.make_set(c) for c in contents]
    wl, wbl, wbi = oracle_lib.match_prefix_batch(sets, ids, keys, key_off)
    assert np.array_equal(lens.cpu().numpy(), wl)
    assert np.array_equal(bl.cpu().numpy(), wbl)
    assert np.array_equal(bi.cpu().numpy(), wbi)


def test_packed_best_combines_like_one_batch(kvx, oracle_lib):
    """Instances spread over 'GPUs': element-wise MAX of per-instance packed
    words (what all-reduce(MAX) does) == the multi-instance batched result."""
    rng = np.random.default_rng(31)
    reqs = _forest(rng, 200, 6, 0, 300)
    key_off = np.concatenate([[0], np.cumsum([len(r) for r in reqs])]).astype(np.int64)
    keys = np.concatenate(reqs).astype(np.int64)
    contents = [np.concatenate([reqs[j][: int(rng.integers(0, len(reqs[j]) + 1))]
                                for j in rng.choice(len(reqs), 15, replace=False)])
                for _ in range(5)]
    ids = [4, 0, 3, 1, 2]
    idx = [_index(kvx, c) for c in contents]
    k, ko = _t(keys, torch.int64), _t(key_off, torch.int64)
    _, bl, bi = kvx.match_prefix_batch(idx, ids, k, ko, want_lens=False)
    packed = torch.stack([kvx.kvx.match_prefix_packed([ix], [i], k, ko) for ix, i in zip(idx, ids)])
    gl, gi = kvx.kvx.best_unpack(packed.max(dim=0).values)
    assert torch.equal(gl, bl) and torch.equal(gi, bi)
    sets = [oracle_lib.make_set(c) for c in contents]
    _, wbl, wbi = oracle_lib.match_prefix_batch(sets, ids, keys, key_off)
    assert np.array_equal(gl.cpu().numpy(), wbl) and np.array_equal(gi.cpu().numpy(), wbi)


def test_index_erase_lookup_growth(kvx, oracle_lib):
    rng = np.random.default_rng(5)
    idx = kvx.BlockIndex(0, 16)  # must grow several times
    keys = rng.integers(-(1 << 62), 1 << 62, size=200_000, dtype=np.int64)
    keys = np.unique(keys)
    rng.shuffle(keys)
    vals = np.arange(len(keys), dtype=np.int64) * 3
    idx.insert(_t(keys, torch.int64), _t(vals, torch.int64))
    st = idx.stats()
    assert st["live"] == len(keys) and st["slots"] >= len(keys) / 0.7
    gone = keys[::2]
    idx.erase(_t(gone, torch.int64))
    idx.erase(_t(gone[:10], torch.int64))  # erasing twice is a no-op
    got = idx.lookup(_t(keys, torch.int64)).cpu().numpy()
    want = vals.copy()
    want[::2] = -1
    assert np.array_equal(got, want)
    assert idx.stats()["live"] == len(keys) - len(gone)
    # re-insert erased keys past their tombstones, then compact
    idx.insert(_t(gone, torch.int64), _t(np.full(len(gone), 7), torch.int64))
    got = idx.lookup(_t(gone, torch.int64)).cpu().numpy()
    assert (got == 7).all()
    idx.reserve(0)
    st = idx.stats()
    assert st["live"] == len(keys) and st["tombstones"] == 0
    got = idx.lookup(_t(keys[1::2], torch.int64)).cpu().numpy()
    assert np.array_equal(got, vals[1::2])
    idx.clear()
    assert idx.stats()["live"] == 0
    assert (idx.lookup(_t(keys[:100], torch.int64)).cpu().numpy() == -1).all()


def test_reserved_keys_never_resident(kvx):
    e, t = kvx.kvx.KEY_EMPTY, kvx.kvx.KEY_TOMBSTONE
    idx = _index(kvx, [5, 6, e, t, 7])
    assert idx.stats()["rejected"] == 2 and idx.stats()["live"] == 3
    idx.erase(_t([6], torch.int64))  # leaves a tombstone: a TOMBSTONE query must not hit it
    for chain, want in [([5, t, 7], 1), ([5, e], 1), ([t], 0), ([5, 7], 2), ([6], 0)]:
        lens, _, _ = kvx.match_prefix_batch([idx], [0], _t(chain, torch.int64),
                                            _t([0, len(chain)], torch.int64))
        assert lens.item() == want, chain


def test_match_long_requests_and_empty(kvx, oracle_lib):
    rng = np.random.default_rng(17)
    chain = rng.integers(0, 1 << 62, size=20000, dtype=np.int64)
    idx = _index(kvx, chain[:19000])
    reqs = [chain, chain[:0], chain[:63], chain[:64], chain[:65], chain[:19000], chain[18999:]]
    key_off = np.concatenate([[0], np.cumsum([len(r) for r in reqs])]).astype(np.int64)
    lens, bl, bi = kvx.match_prefix_batch([idx], [9], _t(np.concatenate(reqs), torch.int64),
                                          _t(key_off, torch.int64))
    assert lens[:, 0].cpu().tolist() == [19000, 0, 63, 64, 65, 19000, 1]
    assert bi.cpu().tolist() == [9] * len(reqs)


def test_block_hash_dispatch_paths(kvx, oracle_lib, monkeypatch):
    """The bs % 16 == 0 kernel with the longest-first order, in index order
    (batches above the order limit), and the any-alignment kernel that a
    token pointer off 16 bytes falls back to: all bit-identical."""
    rng = np.random.default_rng(5)
    lens = rng.integers(0, 3000, size=300)
    lens[7] = 0
    tok_off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    tokens = rng.integers(0, 32000, size=int(tok_off[-1]) + 8).astype(np.int32)
    want, _ = oracle_lib.block_hash_batch(tokens, tok_off, 32)
    t = _t(tokens, torch.int32)
    off = _t(tok_off, torch.int64)
    keys, _ = kvx.chain_hash_batch(t, off, 32)
    assert np.array_equal(keys.cpu().numpy(), want)
    monkeypatch.setenv("KVX_HASH_ORDER_MAX", "10")  # 300 requests > 10: index order
    keys, _ = kvx.chain_hash_batch(t, off, 32)
    assert np.array_equal(keys.cpu().numpy(), want)
    monkeypatch.delenv("KVX_HASH_ORDER_MAX")
    # token pointer 4 bytes past a 16-byte boundary: the fused any-alignment kernel
    big = _t(np.concatenate([[0], tokens]), torch.int32)
    keys, _ = kvx.chain_hash_batch(big[1:], off, 32)
    assert np.array_equal(keys.cpu().numpy(), want)
    monkeypatch.setenv("KVX_HASH_KERNEL", "fused")
    keys, _ = kvx.chain_hash_batch(t, off, 32)
    assert np.array_equal(keys.cpu().numpy(), want)


def test_block_hash_concurrent_streams(kvx, oracle_lib):
    """Two batches in flight on two streams of one device (their claim
    counters and orders must not be shared): both bit-exact."""
    rng = np.random.default_rng(11)
    batches = []
    for n in (500, 700):
        lens = rng.integers(0, 4000, size=n)
        tok_off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        tokens = rng.integers(0, 32000, size=int(tok_off[-1])).astype(np.int32)
        want, _ = oracle_lib.block_hash_batch(tokens, tok_off, 16)
        batches.append((_t(tokens, torch.int32), _t(tok_off, torch.int64), want))
    streams = [torch.cuda.Stream(DEV), torch.cuda.Stream(DEV)]
    torch.cuda.synchronize()
    outs = []
    for _ in range(3):
        for (t, off, _w), st in zip(batches, streams):
            outs.append(kvx.chain_hash_batch(t, off, 16, stream=st)[0])
    torch.cuda.synchronize()
    for i, k in enumerate(outs):
        assert np.array_equal(k.cpu().numpy(), batches[i % 2][2])


def test_config4_scale_match_vs_oracle(kvx, oracle_lib):
    """Config 4 scale: 1M-key instance indices (two instances, Zipf sessions,
    8K-24K-token requests), the whole batch hashed and matched on the GPU;
    every per-instance length and every (best_len, best_id) equals the C
    restatement over the same key sets (kvcache.cpp:150-154,
    conductor.cpp:57-73)."""
    from paper_2407_00079_b200.workloads import MatchWorkload
    mw = MatchWorkload(n_req=1024).build()
    keys, ko = kvx.chain_hash_batch(_t(mw.tokens, torch.int32), _t(mw.tok_off, torch.int64),
                                    mw.block_size)
    wkeys, wko = kvx.chain_hash_batch(_t(mw.warm_tokens, torch.int32),
                                      _t(mw.warm_tok_off, torch.int64), mw.block_size)
    wk, wo = wkeys.cpu().numpy(), wko.cpu().numpy()
    n_sess = len(mw.session_ids)
    contents = []
    for inst in range(2):
        own = np.concatenate([wk[wo[j]:wo[j + 1]] for j in range(n_sess) if j % 2 == inst])
        own = own[: mw.pool_keys]
        contents.append(np.concatenate([own, mw.filler_keys(mw.pool_keys - len(own), inst)]))
    idx = [_index(kvx, c) for c in contents]
    assert all(ix.stats()["live"] == mw.pool_keys for ix in idx)
    ids = [7, 2]
    lens, bl, bi = kvx.match_prefix_batch(idx, ids, keys, ko)
    k_ref, ko_ref = oracle_lib.block_hash_batch(mw.tokens, mw.tok_off, mw.block_size)
    assert np.array_equal(keys.cpu().numpy(), k_ref)
    sets = [oracle_lib.make_set(c) for c in contents]
    wl, wbl, wbi = oracle_lib.match_prefix_batch(sets, ids, k_ref, ko_ref)
    for h in sets:
        oracle_lib.free_set(h)
    assert wbl.sum() > 0 and (wbl > 0).mean() > 0.5  # the sessions' earlier turns are found
    assert np.array_equal(lens.cpu().numpy(), wl)
    assert np.array_equal(bl.cpu().numpy(), wbl)
    assert np.array_equal(bi.cpu().numpy(), wbi)


@pytest.mark.parametrize("bs,n_inst,n_req", [(16, 1, 300), (16, 3, 300), (32, 2, 97), (5, 2, 60),
                                             (16, 1, 40000)])
def test_hash_match_fused_equals_two_calls(kvx, oracle_lib, bs, n_inst, n_req):
    """kvx_hash_match_batch (the match of each request started by the hash's
    completion queue) == kvx_chain_hash_batch + kvx_match_prefix_batch, and
    == the oracle; ragged, empty and sub-block requests included; bs=5 runs
    the sequential fallback."""
    rng = np.random.default_rng(bs * 100 + n_inst)
    hi = 30 * bs if n_req < 1000 else 60
    lens = rng.integers(0, hi, size=n_req)
    lens[:3] = [0, 1, bs]
    tok_off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    tokens = rng.integers(0, 32000, size=int(tok_off[-1]) + 8).astype(np.int32)
    want_keys, wko = oracle_lib.block_hash_batch(tokens, tok_off, bs)
    contents = []
    for i in range(n_inst):  # each instance holds random prefixes of some requests' chains
        pick = rng.choice(n_req, size=min(n_req, 50), replace=False)
        ks = [want_keys[wko[p]: wko[p] + int(rng.integers(0, wko[p + 1] - wko[p] + 1))] for p in pick]
        ks.append(rng.integers(0, 1 << 62, size=20, dtype=np.int64))
        contents.append(np.concatenate(ks).astype(np.int64))
    ids = [5 - 2 * i for i in range(n_inst)]
    idx = [_index(kvx, c) for c in contents]
    keys, ko, lens_out, bl, bi = kvx.kvx.hash_match_batch(
        _t(tokens, torch.int32), _t(tok_off, torch.int64), bs, idx, ids, want_lens=True)
    torch.cuda.synchronize()
    assert np.array_equal(keys.cpu().numpy(), want_keys)
    sets = [oracle_lib.make_set(c) for c in contents]
    wl, wbl, wbi = oracle_lib.match_prefix_batch(sets, ids, want_keys, wko)
    assert np.array_equal(lens_out.cpu().numpy(), wl)
    assert np.array_equal(bl.cpu().numpy(), wbl)
    assert np.array_equal(bi.cpu().numpy(), wbi)
    # repeated calls on the same stream reuse the completion queue
    keys2, _, _, bl2, bi2 = kvx.kvx.hash_match_batch(
        _t(tokens, torch.int32), _t(tok_off, torch.int64), bs, idx, ids)
    torch.cuda.synchronize()
    assert np.array_equal(keys2.cpu().numpy(), want_keys)
    assert np.array_equal(bl2.cpu().numpy(), wbl) and np.array_equal(bi2.cpu().numpy(), wbi)
