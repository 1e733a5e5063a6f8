"""ctypes bindings for the CPU oracle (TEST INFRASTRUCTURE ONLY; see __init__)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libkvref.so")

_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)
_u8p = C.POINTER(C.c_uint8)

__all__ = ["Oracle", "RefLib", "ref_available", "build_oracle", "POLICY"]

POLICY = {"lru": 0, "lfu": 1, "length_aware": 2}


def build_oracle(ref: bool = False) -> None:
    """Compile liboracle.so (and _ref/libkvref.so when /root/reference exists)."""
    target = ["all"] if ref else [LIB_PATH]
    subprocess.run(["make", "-s", "-C", HERE, *target], check=True)


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t) if a is not None else None


class Oracle:
    """Plain-C restatement (kvx_oracle.c)."""

    def __init__(self):
        if not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(
            os.path.join(HERE, "kvx_oracle.c")
        ):
            build_oracle(ref=False)
        L = C.CDLL(LIB_PATH)
        self.L = L
        L.kvo_chain_hash.restype = C.c_int64
        L.kvo_chain_hash.argtypes = [C.c_int64, C.c_uint64]
        L.kvo_content_hash.restype = C.c_uint64
        L.kvo_content_hash.argtypes = [_i32p, C.c_int64]
        L.kvo_block_hash_batch.restype = None
        L.kvo_block_hash_batch.argtypes = [_i32p, _i64p, C.c_int64, C.c_int64, _i64p, _i64p]
        L.kvo_set_create.restype = C.c_void_p
        L.kvo_set_create.argtypes = [_i64p, C.c_int64]
        L.kvo_set_destroy.argtypes = [C.c_void_p]
        L.kvo_set_contains.restype = C.c_int
        L.kvo_set_contains.argtypes = [C.c_void_p, C.c_int64]
        L.kvo_match_prefix.restype = C.c_int64
        L.kvo_match_prefix.argtypes = [C.c_void_p, _i64p, C.c_int64]
        L.kvo_match_prefix_batch.restype = None
        L.kvo_match_prefix_batch.argtypes = [C.POINTER(C.c_void_p), _i32p, C.c_int64, _i64p,
                                             _i64p, C.c_int64, _i64p, _i64p, _i32p]
        for fn in ("kvo_gather", "kvo_scatter"):
            getattr(L, fn).restype = None
        L.kvo_gather.argtypes = [C.c_void_p, C.c_int64, C.c_int64, _i32p, C.c_int64, C.c_int64,
                                 C.c_int64, C.c_void_p, C.c_int]
        L.kvo_scatter.argtypes = [C.c_void_p, C.c_int64, C.c_int64, _i32p, C.c_int64, C.c_int64,
                                  C.c_int64, C.c_void_p, C.c_int]
        L.kvo_copy_paged.restype = None
        L.kvo_copy_paged.argtypes = [C.c_void_p, C.c_int64, _i32p, C.c_void_p, C.c_int64, _i32p,
                                     C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int]
        L.kvo_mix64.restype = C.c_uint64
        L.kvo_mix64.argtypes = [C.c_uint64]
        L.kvo_slab_seed.restype = C.c_uint64
        L.kvo_slab_seed.argtypes = [C.c_uint32] * 4
        L.kvo_kv_word.restype = C.c_uint64
        L.kvo_kv_word.argtypes = [C.c_uint64, C.c_uint64]
        L.kvo_fill_pool.restype = None
        L.kvo_fill_pool.argtypes = [C.c_void_p, C.c_uint32, C.c_int64, C.c_int64, C.c_int64,
                                    C.c_int]
        L.kvo_alloc_lowest_free.restype = C.c_int64
        L.kvo_alloc_lowest_free.argtypes = [_u8p, C.c_int64, C.c_int64, _i32p]

    # ---- hashing -------------------------------------------------------
    def chain_hash(self, prev: int, content: int) -> int:
        return int(self.L.kvo_chain_hash(int(prev), int(content) & 0xFFFFFFFFFFFFFFFF))

    def content_hash(self, tokens) -> int:
        t = np.ascontiguousarray(tokens, dtype=np.int32)
        return int(self.L.kvo_content_hash(_p(t, _i32p), len(t)))

    @staticmethod
    def key_offsets(tok_off: np.ndarray, bs: int) -> np.ndarray:
        lens = np.diff(np.asarray(tok_off, dtype=np.int64))
        blocks = (lens + bs - 1) // bs
        return np.concatenate([[0], np.cumsum(blocks)]).astype(np.int64)

    def block_hash_batch(self, tokens, tok_off, bs: int):
        t = np.ascontiguousarray(tokens, dtype=np.int32)
        to = np.ascontiguousarray(tok_off, dtype=np.int64)
        ko = self.key_offsets(to, bs)
        keys = np.zeros(int(ko[-1]), dtype=np.int64)
        self.L.kvo_block_hash_batch(_p(t, _i32p), _p(to, _i64p), len(to) - 1, bs, _p(ko, _i64p),
                                    _p(keys, _i64p))
        return keys, ko

    # ---- match ---------------------------------------------------------
    def make_set(self, keys):
        k = np.ascontiguousarray(keys, dtype=np.int64)
        return self.L.kvo_set_create(_p(k, _i64p), len(k))

    def free_set(self, s):
        self.L.kvo_set_destroy(s)

    def match_prefix(self, s, keys) -> int:
        k = np.ascontiguousarray(keys, dtype=np.int64)
        return int(self.L.kvo_match_prefix(s, _p(k, _i64p), len(k)))

    def match_prefix_batch(self, sets, inst_ids, keys, key_off):
        n_inst = len(sets)
        arr = (C.c_void_p * n_inst)(*sets)
        ids = np.ascontiguousarray(inst_ids, dtype=np.int32)
        k = np.ascontiguousarray(keys, dtype=np.int64)
        ko = np.ascontiguousarray(key_off, dtype=np.int64)
        n_req = len(ko) - 1
        lens = np.zeros(n_req * n_inst, dtype=np.int64)
        bl = np.zeros(n_req, dtype=np.int64)
        bi = np.zeros(n_req, dtype=np.int32)
        self.L.kvo_match_prefix_batch(arr, _p(ids, _i32p), n_inst, _p(k, _i64p), _p(ko, _i64p),
                                      n_req, _p(lens, _i64p), _p(bl, _i64p), _p(bi, _i32p))
        return lens.reshape(n_req, n_inst), bl, bi

    # ---- bytes ---------------------------------------------------------
    def gather(self, pool: np.ndarray, slots: int, slab: int, src_table, layer_lo, layer_hi,
               buf: np.ndarray, nthreads: int = 1):
        t = np.ascontiguousarray(src_table, dtype=np.int32)
        self.L.kvo_gather(pool.ctypes.data, slots, slab, _p(t, _i32p), len(t), layer_lo,
                          layer_hi, buf.ctypes.data, nthreads)

    def scatter(self, pool: np.ndarray, slots: int, slab: int, dst_table, layer_lo, layer_hi,
                buf: np.ndarray, nthreads: int = 1):
        t = np.ascontiguousarray(dst_table, dtype=np.int32)
        self.L.kvo_scatter(pool.ctypes.data, slots, slab, _p(t, _i32p), len(t), layer_lo,
                           layer_hi, buf.ctypes.data, nthreads)

    def copy_paged(self, src_pool, src_slots, src_table, dst_pool, dst_slots, dst_table, slab,
                   layer_lo, layer_hi, nthreads: int = 1):
        st = np.ascontiguousarray(src_table, dtype=np.int32)
        dt = np.ascontiguousarray(dst_table, dtype=np.int32)
        assert len(st) == len(dt)
        self.L.kvo_copy_paged(src_pool.ctypes.data, src_slots, _p(st, _i32p), dst_pool.ctypes.data,
                              dst_slots, _p(dt, _i32p), slab, len(st), layer_lo, layer_hi,
                              nthreads)

    def fill_pool(self, pool: np.ndarray, pool_id: int, layers: int, slots: int, slab: int,
                  nthreads: int = 1):
        assert pool.nbytes >= layers * 2 * slots * slab
        self.L.kvo_fill_pool(pool.ctypes.data, pool_id, layers, slots, slab, nthreads)

    def slab_seed(self, pool_id, layer, kv, slot) -> int:
        return int(self.L.kvo_slab_seed(pool_id, layer, kv, slot))

    def kv_word(self, seed, word) -> int:
        return int(self.L.kvo_kv_word(seed, word))

    def mix64(self, z) -> int:
        return int(self.L.kvo_mix64(z & 0xFFFFFFFFFFFFFFFF))

    def alloc_lowest_free(self, used: np.ndarray, n: int):
        out = np.zeros(max(n, 1), dtype=np.int32)
        got = self.L.kvo_alloc_lowest_free(_p(used, _u8p), len(used), n, _p(out, _i32p))
        return int(got), out[:n]


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


class RefLib:
    """The reference's own kvcache/conductor/perf_model, compiled in place."""

    def __init__(self):
        if not ref_available():
            raise FileNotFoundError(REF_PATH)
        L = C.CDLL(REF_PATH)
        self.L = L
        L.kvref_chain_hash.restype = C.c_int64
        L.kvref_chain_hash.argtypes = [C.c_int64, C.c_uint64]
        L.kvref_pool_create.restype = C.c_void_p
        L.kvref_pool_create.argtypes = [C.c_int64, C.c_int]
        L.kvref_pool_destroy.argtypes = [C.c_void_p]
        L.kvref_pool_admit.restype = C.c_int64
        L.kvref_pool_admit.argtypes = [C.c_void_p, _i64p, C.c_int64, C.c_int64, C.c_int64, _i64p,
                                       C.c_int64, _i64p, _i64p, _i32p]
        L.kvref_pool_insert_replicated.restype = C.c_int64
        L.kvref_pool_insert_replicated.argtypes = [C.c_void_p, _i64p, C.c_int64, C.c_int64,
                                                   _i64p, C.c_int64]
        L.kvref_pool_match_prefix.restype = C.c_int64
        L.kvref_pool_match_prefix.argtypes = [C.c_void_p, _i64p, C.c_int64]
        L.kvref_pool_contains.restype = C.c_int
        L.kvref_pool_contains.argtypes = [C.c_void_p, C.c_int64]
        L.kvref_pool_size.restype = C.c_int64
        L.kvref_pool_size.argtypes = [C.c_void_p]
        L.kvref_pool_stats.restype = None
        L.kvref_pool_stats.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.kvref_find_best_prefix_match.restype = C.c_int
        L.kvref_find_best_prefix_match.argtypes = [C.POINTER(C.c_void_p), _i32p, C.c_int64, _i64p,
                                                   C.c_int64, _i64p, _i32p]
        L.kvref_match_batch_mt.restype = None
        L.kvref_match_batch_mt.argtypes = [C.POINTER(C.c_void_p), _i32p, C.c_int64, _i64p, _i64p,
                                           C.c_int64, _i64p, _i32p, C.c_int]
        L.kvref_block_hash_mt.restype = None
        L.kvref_block_hash_mt.argtypes = [_i32p, _i64p, C.c_int64, C.c_int64, _i64p, _i64p,
                                          C.c_int]
        L.kvref_pool_insert_many.restype = None
        L.kvref_pool_insert_many.argtypes = [C.c_void_p, _i64p, C.c_int64]
        L.kvref_estimate_transfer_time.restype = C.c_double
        L.kvref_estimate_transfer_time.argtypes = [C.c_int64, C.c_double, C.c_double,
                                                   C.c_double, C.c_double]

    def chain_hash(self, prev: int, content: int) -> int:
        return int(self.L.kvref_chain_hash(int(prev), int(content) & 0xFFFFFFFFFFFFFFFF))

    def schedule(self, perf8, chunk, stages, l_ttft, l_tbt, threshold, block_size, now, pools,
                 ids, busy, sender, queued, dids, dbatch, dkv, input_len, keys):
        """kvref::schedule(kKvcacheCentric) for one request -> (ints[9], doubles[5])."""
        f = self.L.kvref_schedule
        if not getattr(f, "_typed", False):
            d, i64, i32 = C.POINTER(C.c_double), _i64p, _i32p
            f.restype = C.c_int
            f.argtypes = [d, C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_double, C.c_int64,
                          C.c_double, C.POINTER(C.c_void_p), i32, d, d, d, C.c_int64, i32, i64,
                          i64, C.c_int64, C.c_int64, i64, C.c_int64, i64, d]
            f._typed = True
        a = lambda x, t: np.ascontiguousarray(x, dtype=t)  # noqa: E731
        pf, b, s, q = (a(perf8, np.float64), a(busy, np.float64), a(sender, np.float64),
                       a(queued, np.float64))
        ii, di, db, dk, k = (a(ids, np.int32), a(dids, np.int32), a(dbatch, np.int64),
                             a(dkv, np.int64), a(keys, np.int64))
        arr = (C.c_void_p * len(pools))(*[p.h for p in pools])
        oi = np.zeros(9, dtype=np.int64)
        od = np.zeros(5, dtype=np.float64)
        dp = C.POINTER(C.c_double)
        rc = f(pf.ctypes.data_as(dp), chunk, stages, l_ttft, l_tbt, threshold, block_size, now, arr,
               _p(ii, _i32p), b.ctypes.data_as(dp), s.ctypes.data_as(dp), q.ctypes.data_as(dp),
               len(pools), _p(di, _i32p), _p(db, _i64p), _p(dk, _i64p), len(di), input_len,
               _p(k, _i64p), len(k), _p(oi, _i64p), od.ctypes.data_as(dp))
        if rc != 0:
            raise ValueError("ValidationError")
        return oi, od

    def pool(self, capacity=None, policy="lru"):
        return RefPool(self, capacity, policy)

    def find_best_prefix_match(self, pools, ids, keys):
        arr = (C.c_void_p * len(pools))(*[p.h for p in pools])
        i = np.ascontiguousarray(ids, dtype=np.int32)
        k = np.ascontiguousarray(keys, dtype=np.int64)
        bl = C.c_int64(0)
        bi = C.c_int32(0)
        rc = self.L.kvref_find_best_prefix_match(arr, _p(i, _i32p), len(pools), _p(k, _i64p),
                                                 len(k), C.byref(bl), C.byref(bi))
        if rc != 0:
            raise ValueError("ValidationError: empty prefill pool")
        return int(bl.value), int(bi.value)

    def block_hash_mt(self, tokens, tok_off, bs, key_off, keys_out, nthreads):
        t = np.ascontiguousarray(tokens, dtype=np.int32)
        to = np.ascontiguousarray(tok_off, dtype=np.int64)
        ko = np.ascontiguousarray(key_off, dtype=np.int64)
        self.L.kvref_block_hash_mt(_p(t, _i32p), _p(to, _i64p), len(to) - 1, bs, _p(ko, _i64p),
                                   _p(keys_out, _i64p), nthreads)
        return keys_out

    def match_batch_mt(self, pools, ids, keys, key_off, nthreads):
        arr = (C.c_void_p * len(pools))(*[p.h for p in pools])
        i = np.ascontiguousarray(ids, dtype=np.int32)
        k = np.ascontiguousarray(keys, dtype=np.int64)
        ko = np.ascontiguousarray(key_off, dtype=np.int64)
        n_req = len(ko) - 1
        bl = np.zeros(n_req, dtype=np.int64)
        bi = np.zeros(n_req, dtype=np.int32)
        self.L.kvref_match_batch_mt(arr, _p(i, _i32p), len(pools), _p(k, _i64p), _p(ko, _i64p),
                                    n_req, _p(bl, _i64p), _p(bi, _i32p), nthreads)
        return bl, bi


class RefPool:
    def __init__(self, lib: RefLib, capacity, policy):
        self.lib = lib
        self.h = lib.L.kvref_pool_create(-1 if capacity is None else int(capacity),
                                         POLICY[policy])
        if not self.h:
            raise ValueError("ValidationError: cache capacity must be >= 1 block")

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.L.kvref_pool_destroy(self.h)
            self.h = None

    def admit_and_touch(self, keys, skip_begin=0, skip_end=0):
        k = np.ascontiguousarray(keys, dtype=np.int64)
        cap = len(k) + self.size() + 1
        ev = np.zeros(cap, dtype=np.int64)
        hits = C.c_int64(0)
        misses = C.c_int64(0)
        trunc = C.c_int32(0)
        n_ev = self.lib.L.kvref_pool_admit(self.h, _p(k, _i64p), len(k), skip_begin, skip_end,
                                           _p(ev, _i64p), cap, C.byref(hits), C.byref(misses),
                                           C.byref(trunc))
        return {"evicted": ev[:n_ev].tolist(), "hits": hits.value, "misses": misses.value,
                "truncated": bool(trunc.value)}

    def insert_replicated(self, keys, chain_offset=0):
        k = np.ascontiguousarray(keys, dtype=np.int64)
        cap = len(k) + self.size() + 1
        ev = np.zeros(cap, dtype=np.int64)
        n_ev = self.lib.L.kvref_pool_insert_replicated(self.h, _p(k, _i64p), len(k), chain_offset,
                                                       _p(ev, _i64p), cap)
        return ev[:n_ev].tolist()

    def insert_many(self, keys):
        k = np.ascontiguousarray(keys, dtype=np.int64)
        self.lib.L.kvref_pool_insert_many(self.h, _p(k, _i64p), len(k))

    def match_prefix(self, keys) -> int:
        k = np.ascontiguousarray(keys, dtype=np.int64)
        return int(self.lib.L.kvref_pool_match_prefix(self.h, _p(k, _i64p), len(k)))

    def contains(self, key) -> bool:
        return bool(self.lib.L.kvref_pool_contains(self.h, int(key)))

    def size(self) -> int:
        return int(self.lib.L.kvref_pool_size(self.h))

    def stats(self):
        h = C.c_uint64(0)
        m = C.c_uint64(0)
        self.lib.L.kvref_pool_stats(self.h, C.byref(h), C.byref(m))
        return int(h.value), int(m.value)
