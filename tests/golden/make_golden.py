"""Generate tests/golden/*.npz from the REFERENCE implementation.

Run in the build container (needs oracle/_ref/libkvref.so, i.e. the reference's
own proj/src/{kvcache,conductor,perf_model}.cpp compiled in place by
oracle/Makefile).  The fixtures are committed so the GPU box -- which has no
/root/reference -- can check both the C restatement and the CUDA path against
the reference's own outputs.

    python tests/golden/make_golden.py

Every expected value below comes from a kvref:: call (chain_hash,
CachePool::match_prefix / admit_and_touch / insert_replicated,
find_best_prefix_match); inputs come from a seeded numpy Generator.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import RefLib, build_oracle, ref_available  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
I64_MIN = -(1 << 63)
I64_MAX = (1 << 63) - 1


def chain_hash_fixture(ref: RefLib) -> None:
    rng = np.random.default_rng(20240700)
    prev = [0, 0, 1, 0, 0, 0, -1, I64_MAX, I64_MIN, 1 << 40, -(1 << 40)]
    content = [1, 2, 1, 3, 4, 0, 0xFFFFFFFFFFFFFFFF, 0, 0xFFFFFFFFFFFFFFFF, 5, 7]
    prev += rng.integers(I64_MIN, I64_MAX, size=500, dtype=np.int64, endpoint=True).tolist()
    content += rng.integers(0, 1 << 64, size=500, dtype=np.uint64).tolist()
    # fold prev=0, content=1..4 is a chain, add it explicitly
    fold = []
    k = 0
    for c in (1, 2, 3, 4):
        k = ref.chain_hash(k, c)
        fold.append(k)
    out = [ref.chain_hash(p, c) for p, c in zip(prev, content)]
    np.savez_compressed(
        os.path.join(OUT, "chain_hash.npz"),
        prev=np.array(prev, dtype=np.int64),
        content=np.array(content, dtype=np.uint64),
        out=np.array(out, dtype=np.int64),
        fold_1_4=np.array(fold, dtype=np.int64),
    )


def block_hash_fixture(ref: RefLib) -> None:
    """Build-defined content hash composed of the reference chain_hash:
    content_i = fold(chain_hash, tokens of block i, from 0);
    key_i = chain_hash(key_{i-1}, content_i), key_{-1} = 0."""
    rng = np.random.default_rng(7)
    cases = {}
    for bs in (1, 5, 16, 64):
        lens = [0, 1, bs - 1 if bs > 1 else 1, bs, bs + 1, 3 * bs, 3 * bs + 2] + rng.integers(
            0, 6 * bs, size=9).tolist()
        # shared-prefix requests: request j copies a prefix of request j-1
        toks = []
        for j, n in enumerate(lens):
            t = rng.integers(0, 32000, size=n).astype(np.int32)
            if j > 0 and len(toks[-1]) > 0 and n > 0:
                share = min(n, len(toks[-1])) // 2
                t[:share] = toks[-1][:share]
            toks.append(t)
        tok_off = np.concatenate([[0], np.cumsum([len(t) for t in toks])]).astype(np.int64)
        tokens = np.concatenate(toks).astype(np.int32) if tok_off[-1] else np.zeros(0, np.int32)
        keys = []
        for t in toks:
            key = 0
            for s in range(0, len(t), bs):
                c = 0
                for tok in t[s:s + bs]:
                    c = ref.chain_hash(c, int(np.uint32(tok)))
                key = ref.chain_hash(key, c & 0xFFFFFFFFFFFFFFFF)
                keys.append(key)
        cases[f"bs{bs}_tokens"] = tokens
        cases[f"bs{bs}_tok_off"] = tok_off
        cases[f"bs{bs}_keys"] = np.array(keys, dtype=np.int64)
    np.savez_compressed(os.path.join(OUT, "block_hash.npz"), **cases)


def match_fixture(ref: RefLib) -> None:
    """Randomized scheduling states in the shape of acceptance criterion 4's
    make_random_state (proj/tests/acceptance_main.cpp:237-302): 2-16 instances,
    each warmed with a random-depth prefix of the query chain plus noise ids;
    expected per-instance match_prefix and find_best_prefix_match from kvref."""
    rng = np.random.default_rng(4004)
    S = 400
    inst_keys, inst_off, inst_cnt = [], [0], []
    q_keys, q_off = [], [0]
    lens, best_len, best_id, inst_ids = [], [], [], []
    for s in range(S):
        blocks = int(rng.integers(1, 25)) if s % 10 else int(rng.integers(1, 200))
        chain = (np.arange(blocks, dtype=np.int64) * 7919 + s * 100000) if s % 3 else \
            rng.integers(I64_MIN + 2, I64_MAX, size=blocks, dtype=np.int64)
        n_inst = int(rng.integers(1, 17))
        pools, ids = [], []
        # instance ids are a permutation so the lowest-id tie-break is not positional
        perm = rng.permutation(n_inst).astype(np.int32) + int(rng.integers(0, 3))
        for i in range(n_inst):
            warm = int(rng.integers(0, blocks + 1))
            noise = rng.integers(10**12, 10**12 + 100, size=int(rng.integers(0, 7)))
            hole = int(rng.integers(0, blocks)) if rng.random() < 0.2 else -1
            content = [int(x) for j, x in enumerate(chain[:warm]) if j != hole]
            # occasionally hold a LATER block without the earlier one (first-miss rule)
            if rng.random() < 0.3 and blocks > warm + 1:
                content.append(int(chain[int(rng.integers(warm + 1, blocks))]))
            content += [int(x) for x in noise]
            p = ref.pool(None, "lru")
            if content:
                p.insert_replicated(np.array(content, dtype=np.int64))
            pools.append(p)
            ids.append(int(perm[i]))
            inst_keys.extend(content)
            inst_off.append(len(inst_keys))
            lens.append(p.match_prefix(chain))
        inst_cnt.append(n_inst)
        inst_ids.extend(ids)
        bl, bi = ref.find_best_prefix_match(pools, ids, chain)
        best_len.append(bl)
        best_id.append(bi)
        q_keys.extend(chain.tolist())
        q_off.append(len(q_keys))
    np.savez_compressed(
        os.path.join(OUT, "match_states.npz"),
        inst_keys=np.array(inst_keys, dtype=np.int64),
        inst_off=np.array(inst_off, dtype=np.int64),
        inst_cnt=np.array(inst_cnt, dtype=np.int64),
        inst_ids=np.array(inst_ids, dtype=np.int32),
        q_keys=np.array(q_keys, dtype=np.int64),
        q_off=np.array(q_off, dtype=np.int64),
        lens=np.array(lens, dtype=np.int64),
        best_len=np.array(best_len, dtype=np.int64),
        best_id=np.array(best_id, dtype=np.int32),
    )


def random_chain_trace(rng, requests, sessions, max_depth):
    """Same structure as oracle::random_chain_trace (proj/tests/oracles.hpp:285-308),
    driven by numpy instead of kvcsim::Rng."""
    chains = [[] for _ in range(sessions)]
    next_id = 0
    out = []
    for _ in range(requests):
        ch = chains[int(rng.integers(0, sessions))]
        depth = int(rng.integers(1, max_depth + 1))
        while len(ch) < depth:
            ch.append(next_id)
            next_id += 1
        out.append(list(ch[:depth]))
    return out


def cachepool_fixture(ref: RefLib) -> None:
    """Put-side sequences through kvref::CachePool: admit_and_touch (with and
    without skip ranges) and insert_replicated, three policies, several
    capacities.  Records every call's evicted list and counters."""
    rng = np.random.default_rng(1001)
    ops_kind, ops_pool, ops_keys, ops_off, ops_a, ops_b = [], [], [], [0], [], []
    exp_ev, exp_ev_off, exp_hits, exp_misses, exp_trunc, exp_match = [], [0], [], [], [], []
    pool_cfg = []
    pid = 0
    for policy in ("lru", "lfu", "length_aware"):
        for cap in (None, 1, 3, 6, 12, 40):
            trace = random_chain_trace(rng, 120, 5, 10)
            p = ref.pool(cap, policy)
            pool_cfg.append((pid, -1 if cap is None else cap, {"lru": 0, "lfu": 1,
                                                               "length_aware": 2}[policy]))
            for chain in trace:
                keys = np.array(chain, dtype=np.int64)
                r = rng.random()
                if r < 0.15:
                    off = int(rng.integers(0, 4))
                    ev = p.insert_replicated(keys, off)
                    kind, a, b = 1, off, 0
                    hits = misses = trunc = 0
                elif r < 0.3 and len(keys) > 1:
                    sb = int(rng.integers(0, len(keys)))
                    se = int(rng.integers(sb, len(keys) + 1))
                    res = p.admit_and_touch(keys, sb, se)
                    ev, hits, misses, trunc = (res["evicted"], res["hits"], res["misses"],
                                               int(res["truncated"]))
                    kind, a, b = 0, sb, se
                else:
                    res = p.admit_and_touch(keys)
                    ev, hits, misses, trunc = (res["evicted"], res["hits"], res["misses"],
                                               int(res["truncated"]))
                    kind, a, b = 0, 0, 0
                ops_kind.append(kind)
                ops_pool.append(pid)
                ops_keys.extend(chain)
                ops_off.append(len(ops_keys))
                ops_a.append(a)
                ops_b.append(b)
                exp_ev.extend(ev)
                exp_ev_off.append(len(exp_ev))
                exp_hits.append(hits)
                exp_misses.append(misses)
                exp_trunc.append(trunc)
                # probe match_prefix against a fresh random chain of this trace
                probe = np.array(trace[int(rng.integers(0, len(trace)))], dtype=np.int64)
                exp_match.append(p.match_prefix(probe))
                ops_keys_probe = probe  # stored via match_probe arrays below
                match_probe_keys.extend(ops_keys_probe.tolist())
                match_probe_off.append(len(match_probe_keys))
            h, m = p.stats()
            final_stats.append((h, m, p.size()))
            pid += 1
    np.savez_compressed(
        os.path.join(OUT, "cachepool_ops.npz"),
        pool_cfg=np.array(pool_cfg, dtype=np.int64),
        ops_kind=np.array(ops_kind, dtype=np.int64),
        ops_pool=np.array(ops_pool, dtype=np.int64),
        ops_keys=np.array(ops_keys, dtype=np.int64),
        ops_off=np.array(ops_off, dtype=np.int64),
        ops_a=np.array(ops_a, dtype=np.int64),
        ops_b=np.array(ops_b, dtype=np.int64),
        exp_ev=np.array(exp_ev, dtype=np.int64),
        exp_ev_off=np.array(exp_ev_off, dtype=np.int64),
        exp_hits=np.array(exp_hits, dtype=np.int64),
        exp_misses=np.array(exp_misses, dtype=np.int64),
        exp_trunc=np.array(exp_trunc, dtype=np.int64),
        exp_match=np.array(exp_match, dtype=np.int64),
        match_probe_keys=np.array(match_probe_keys, dtype=np.int64),
        match_probe_off=np.array(match_probe_off, dtype=np.int64),
        final_stats=np.array(final_stats, dtype=np.int64),
    )


def schedule_fixture(ref: RefLib) -> None:
    """Randomized cluster snapshots shaped like acceptance criterion 4's
    make_random_state (proj/tests/acceptance_main.cpp:237-302), 4 requests per
    snapshot; expected decisions from kvref::schedule(kKvcacheCentric)."""
    rng = np.random.default_rng(4004)
    S, R = 300, 4
    rows = {k: [] for k in ("perf", "ints", "dbl", "inst_keys", "inst_off", "inst_ids", "busy",
                            "sender", "queued", "n_inst", "dec_ids", "dec_batch", "dec_kv",
                            "n_dec", "req_input", "req_keys", "req_off", "exp_i", "exp_d")}
    rows["inst_off"].append(0)
    rows["req_off"].append(0)
    for s in range(S):
        perf = [0.01 + rng.random() * 0.2, rng.random() * 1e-5, rng.random() * 20.0,
                rng.random() * 2.0, rng.random(), 1000.0 + rng.random() * 2e5,
                1e5 + rng.random() * 1e7, 1e5 + rng.random() * 1e7]
        chunk, stages = int(rng.integers(256, 4097)), int(rng.integers(1, 5))
        threshold = 1.0 + rng.random() * 7.0
        l_ttft = 200.0 + rng.random() * 2000.0 if rng.random() < 0.3 else 1e9
        l_tbt = 5.0 + rng.random() * 50.0 if rng.random() < 0.3 else 1e9
        now = rng.random() * 200.0
        blocks = int(rng.integers(1, 25))
        chain = np.arange(blocks, dtype=np.int64) + s * 1000
        n_inst = int(rng.integers(2, 17))
        ids = rng.permutation(n_inst).astype(np.int32)
        pools = []
        for i in range(n_inst):
            warm = int(rng.integers(0, blocks + 1))
            content = list(chain[:warm]) + [int(x) for x in
                                            900000 + rng.integers(0, 100, int(rng.integers(0, 7)))]
            p = ref.pool(None, "lru")
            if content:
                p.insert_replicated(np.array(content, dtype=np.int64))
            pools.append(p)
            rows["inst_keys"].extend(int(x) for x in content)
            rows["inst_off"].append(len(rows["inst_keys"]))
        busy = [rng.random() * 500.0 if rng.random() < 0.5 else 0.0 for _ in range(n_inst)]
        sender = [rng.random() * 300.0 if rng.random() < 0.5 else 0.0 for _ in range(n_inst)]
        queued = [rng.random() * 1500.0 for _ in range(n_inst)]
        n_dec = int(rng.integers(1, 7))
        dids = rng.permutation(n_dec).astype(np.int32)
        dbatch = rng.integers(0, 33, n_dec)
        dkv = rng.integers(0, 200001, n_dec)
        for _ in range(R):
            nb = int(rng.integers(1, blocks + 1))
            keys = np.concatenate([chain[:nb], 5_000_000 + s * 10 + rng.integers(0, 5, 1)])
            keys = keys[: nb + int(rng.integers(0, 2))]
            inp = len(keys) * 512 - int(rng.integers(0, 512))
            ei, ed = ref.schedule(perf, chunk, stages, l_ttft, l_tbt, threshold, 512, now, pools,
                                  ids, busy, sender, queued, dids, dbatch, dkv, inp, keys)
            rows["req_input"].append(inp)
            rows["req_keys"].extend(int(x) for x in keys)
            rows["req_off"].append(len(rows["req_keys"]))
            rows["exp_i"].append(ei)
            rows["exp_d"].append(ed)
        rows["perf"].append(perf)
        rows["ints"].append([chunk, stages])
        rows["dbl"].append([l_ttft, l_tbt, threshold, now])
        rows["inst_ids"].extend(ids.tolist())
        rows["busy"].extend(busy)
        rows["sender"].extend(sender)
        rows["queued"].extend(queued)
        rows["n_inst"].append(n_inst)
        rows["dec_ids"].extend(dids.tolist())
        rows["dec_batch"].extend(dbatch.tolist())
        rows["dec_kv"].extend(dkv.tolist())
        rows["n_dec"].append(n_dec)
    out = {k: np.array(v) for k, v in rows.items()}
    out["requests_per_state"] = np.array(R)
    np.savez_compressed(os.path.join(OUT, "schedule_states.npz"), **out)


match_probe_keys: list = []
match_probe_off: list = [0]
final_stats: list = []


def main() -> None:
    if not ref_available():
        build_oracle(ref=True)
    ref = RefLib()
    chain_hash_fixture(ref)
    block_hash_fixture(ref)
    match_fixture(ref)
    cachepool_fixture(ref)
    schedule_fixture(ref)
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)), "bytes")


if __name__ == "__main__":
    main()
