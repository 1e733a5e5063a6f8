"""CPU tests: pin the C restatement (oracle/kvx_oracle.c) against the
reference's own outputs (tests/golden, generated from oracle/_ref) and the
reference's known-answer tests (proj/tests/test_kvcache.cpp,
proj/tests/test_conductor.cpp), and pin the build-defined byte stages with
this repo's own KATs."""
import numpy as np
import pytest

from conftest import golden

# SURVEY.md Appendix A, generated from the compiled reference chain_hash.
APPENDIX_A = [
    ((0, 1), 2722740466618122910),
    ((0, 2), 2805327317107431418),
    ((1, 1), 4366858250831754186),
    ((-1, 0xFFFFFFFFFFFFFFFF), 8432741605462336350),
]
FOLD_1_4 = [2722740466618122910, 2073803827775855637, 3042475482000967161,
            2236103413144714628]


def test_chain_hash_appendix_a(oracle_lib):
    for (p, c), want in APPENDIX_A:
        assert oracle_lib.chain_hash(p, c) == want
    k = 0
    for c, want in zip((1, 2, 3, 4), FOLD_1_4):
        k = oracle_lib.chain_hash(k, c)
        assert k == want


def test_chain_hash_golden(oracle_lib):
    g = golden("chain_hash.npz")
    got = [oracle_lib.chain_hash(int(p), int(c)) for p, c in zip(g["prev"], g["content"])]
    assert np.array_equal(np.array(got, dtype=np.int64), g["out"])
    assert g["fold_1_4"].tolist() == FOLD_1_4


def test_chain_hash_properties(oracle_lib):
    # proj/tests/test_kvcache.cpp:30-35
    h = oracle_lib.chain_hash
    assert h(0, 1) == h(0, 1)
    assert h(0, 1) != h(0, 2)
    assert h(0, 1) != h(1, 1)
    assert h(0, 1) >= 0


@pytest.mark.parametrize("bs", [1, 5, 16, 64])
def test_block_hash_golden(oracle_lib, bs):
    g = golden("block_hash.npz")
    keys, ko = oracle_lib.block_hash_batch(g[f"bs{bs}_tokens"], g[f"bs{bs}_tok_off"], bs)
    assert np.array_equal(keys, g[f"bs{bs}_keys"])
    lens = np.diff(g[f"bs{bs}_tok_off"])
    assert np.array_equal(np.diff(ko), (lens + bs - 1) // bs)


def test_block_hash_prefix_property(oracle_lib):
    # equal key i <=> equal tokens [0, (i+1)*bs) (prefix-chained ids, kvcache.hpp:17-19)
    rng = np.random.default_rng(3)
    a = rng.integers(0, 32000, 160).astype(np.int32)
    b = a.copy()
    b[100] += 1  # differs in block 6 (bs=16)
    toks = np.concatenate([a, b])
    keys, ko = oracle_lib.block_hash_batch(toks, np.array([0, 160, 320]), 16)
    ka, kb = keys[:10], keys[10:]
    assert np.array_equal(ka[:6], kb[:6])
    assert not np.any(ka[6:] == kb[6:])


def _kat_sets(o, contents):
    return [o.make_set(np.array(c, dtype=np.int64)) for c in contents]


def test_match_prefix_kats(oracle_lib):
    # proj/tests/test_kvcache.cpp:37-73
    o = oracle_lib
    chain = [1, 2, 3]
    s_empty, s1, s3, sfull = _kat_sets(o, [[], [1], [3], [1, 2, 3]])
    assert o.match_prefix(s_empty, chain) == 0
    assert o.match_prefix(s1, chain) == 1
    assert o.match_prefix(s3, chain) == 0  # stops at the first miss
    assert o.match_prefix(sfull, chain) == 3
    assert o.match_prefix(sfull, []) == 0


def test_find_best_prefix_match_kats(oracle_lib):
    # proj/tests/test_conductor.cpp:81-113
    o = oracle_lib
    chain = np.arange(8, dtype=np.int64)
    sets = _kat_sets(o, [[], []])
    _, bl, bi = o.match_prefix_batch(sets, [0, 1], chain, [0, 8])
    assert (bl[0], bi[0]) == (0, 0)
    sets = _kat_sets(o, [range(3), range(7), range(7)])
    _, bl, bi = o.match_prefix_batch(sets, [0, 1, 2], chain, [0, 8])
    assert (bl[0], bi[0]) == (7, 1)
    sets = _kat_sets(o, [range(2), range(8)])
    _, bl, bi = o.match_prefix_batch(sets, [0, 1], chain, [0, 8])
    assert (bl[0], bi[0]) == (8, 1)


def test_match_states_golden(oracle_lib):
    g = golden("match_states.npz")
    o = oracle_lib
    ii = 0
    for s in range(len(g["inst_cnt"])):
        n_inst = int(g["inst_cnt"][s])
        sets, ids = [], []
        for i in range(n_inst):
            lo, hi = g["inst_off"][ii], g["inst_off"][ii + 1]
            sets.append(o.make_set(g["inst_keys"][lo:hi]))
            ids.append(int(g["inst_ids"][ii]))
            ii += 1
        q = g["q_keys"][g["q_off"][s]:g["q_off"][s + 1]]
        lens, bl, bi = o.match_prefix_batch(sets, ids, q, [0, len(q)])
        base = ii - n_inst
        assert lens[0].tolist() == g["lens"][base:ii].tolist()
        assert (bl[0], bi[0]) == (g["best_len"][s], g["best_id"][s])
        for st in sets:
            o.free_set(st)


def test_oracle_matches_reference_live(oracle_lib, ref_lib):
    """Where the reference is compiled here, cross-check fresh random inputs."""
    rng = np.random.default_rng(99)
    for _ in range(200):
        p = int(rng.integers(-(1 << 63), (1 << 63) - 1, dtype=np.int64))
        c = int(rng.integers(0, 1 << 64, dtype=np.uint64))
        assert oracle_lib.chain_hash(p, c) == ref_lib.chain_hash(p, c)
    chain = np.arange(50, dtype=np.int64)
    pools = []
    sets = []
    for d in (0, 10, 30, 30, 5):
        rp = ref_lib.pool(None, "lru")
        if d:
            rp.insert_replicated(chain[:d])
        pools.append(rp)
        sets.append(oracle_lib.make_set(chain[:d]))
    ids = [4, 3, 2, 1, 0]
    _, bl, bi = oracle_lib.match_prefix_batch(sets, ids, chain, [0, 50])
    assert (int(bl[0]), int(bi[0])) == ref_lib.find_best_prefix_match(pools, ids, chain)
    with pytest.raises(ValueError):
        ref_lib.find_best_prefix_match([], [], chain)


# ---- build-defined byte stages: this repo's own KATs ---------------------

def test_kv_content_kats(oracle_lib):
    o = oracle_lib
    # splitmix64 finalizer of 0 (the well-known first splitmix64 output)
    assert o.mix64(0) == 0xE220A8397B1DCDAF
    s0 = o.slab_seed(0, 0, 0, 0)
    assert s0 == o.mix64(0)
    assert o.slab_seed(1, 0, 0, 0) != o.slab_seed(0, 1, 0, 0)
    assert o.slab_seed(0, 0, 1, 0) != o.slab_seed(0, 0, 0, 1)
    assert o.kv_word(s0, 0) == o.mix64(s0)


def test_fill_gather_scatter_roundtrip(oracle_lib):
    o = oracle_lib
    L, slots, slab = 3, 11, 256
    src = np.zeros(L * 2 * slots * slab, dtype=np.uint8)
    o.fill_pool(src, 7, L, slots, slab, nthreads=2)
    words = src.view(np.uint64).reshape(L, 2, slots, slab // 8)
    seed = o.slab_seed(7, 2, 1, 5)
    assert int(words[2, 1, 5, 3]) == o.kv_word(seed, 3)
    src_table = np.array([4, 0, 9, 9, 2], dtype=np.int32)  # duplicates are legal on the source
    used = np.zeros(13, dtype=np.uint8)
    used[[0, 3]] = 1
    got, dst_table = o.alloc_lowest_free(used, 5)
    assert got == 5 and dst_table.tolist() == [1, 2, 4, 5, 6]
    buf = np.zeros((L - 1) * 2 * 5 * slab, dtype=np.uint8)
    o.gather(src, slots, slab, src_table, 1, 3, buf, nthreads=3)
    dst = np.zeros(L * 2 * 13 * slab, dtype=np.uint8)
    o.scatter(dst, 13, slab, dst_table, 1, 3, buf)
    dw = dst.view(np.uint64).reshape(L, 2, 13, slab // 8)
    for li in (1, 2):
        for kv in (0, 1):
            for b in range(5):
                assert np.array_equal(dw[li, kv, dst_table[b]], words[li, kv, src_table[b]])
    assert not dw[0].any()  # layer 0 not in range
    dst2 = np.zeros_like(dst)
    o.copy_paged(src, slots, src_table, dst2, 13, dst_table, slab, 1, 3, nthreads=2)
    assert np.array_equal(dst, dst2)


def test_alloc_exhaustion(oracle_lib):
    used = np.zeros(4, dtype=np.uint8)
    got, _ = oracle_lib.alloc_lowest_free(used, 5)
    assert got < 5 and not used.any()
