"""Python face of the GPU-backed drop-in block manager (libkvcsim_gpu.so,
include/kvcsim_c.h) -- the reference's ``kvcsim::CachePool`` API
(/root/reference/proj/include/kvcsim/kvcache.hpp:44-102) and
``find_best_prefix_match`` (proj/include/kvcsim/conductor.hpp:63-64), batched.

Method names, argument meaning and error behaviour follow the reference:
capacity 0 and an empty instance list raise ``ValidationError``.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

from .kvx import KVX_EINVAL, KVX_OK, KvxError, ValidationError
from .kvx import alive as _kvx_alive

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libkvcsim_gpu.so")
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} missing: run `make -C {_HERE}/csrc`")
_L = C.CDLL(LIB_PATH)

_vp = C.c_void_p
_i64 = C.c_int64
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)


def _sig(name, res, *args):
    f = getattr(_L, name)
    f.restype = res
    f.argtypes = list(args)


_sig("kvcsim_last_error", C.c_char_p)
_sig("kvcsim_pool_create", C.c_int, _i64, C.c_int, C.POINTER(_vp))
_sig("kvcsim_pool_destroy", None, _vp)
_sig("kvcsim_pool_admit", C.c_int, _vp, _i64p, _i64, _i64, _i64, _i64p, _i64, _i64p, _i64p, _i64p,
     _i32p)
_sig("kvcsim_pool_insert_replicated", C.c_int, _vp, _i64p, _i64, _i64, _i64p, _i64, _i64p)
_sig("kvcsim_pool_match_prefix", C.c_int, _vp, _i64p, _i64, _i64p)
_sig("kvcsim_pool_contains", C.c_int, _vp, _i64, _i32p)
_sig("kvcsim_pool_size", _i64, _vp)
_sig("kvcsim_pool_stats", None, _vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64))
_sig("kvcsim_find_best_prefix_match_batch", C.c_int, C.POINTER(_vp), _i32p, _i64, _i64p, _i64p,
     _i64, _i64p, _i64p, _i32p)

POLICIES = {"lru": 0, "lfu": 1, "length_aware": 2}


def _check(st):
    if st == KVX_OK:
        return
    msg = (_L.kvcsim_last_error() or b"").decode(errors="replace")
    if st == KVX_EINVAL:
        raise ValidationError(msg)
    raise KvxError(st, msg)


def _keys(a):
    k = np.ascontiguousarray(a, dtype=np.int64)
    return k, k.ctypes.data_as(_i64p)


class CachePool:
    """kvcsim::CachePool: host policy state + B200 block index."""

    def __init__(self, capacity: Optional[int] = None, policy: str = "lru"):
        h = _vp()
        _check(_L.kvcsim_pool_create(-1 if capacity is None else int(capacity),
                                     POLICIES[policy], C.byref(h)))
        self.h = h
        self.capacity = capacity
        self.policy = policy

    def close(self):
        if getattr(self, "h", None) and _kvx_alive():
            _L.kvcsim_pool_destroy(self.h)
            self.h = None

    __del__ = close

    def admit_and_touch(self, blocks, skip_begin: int = 0, skip_end: int = 0) -> dict:
        k, kp = _keys(blocks)
        cap = len(k) + self.size() + 1
        ev = np.zeros(cap, dtype=np.int64)
        n_ev, hits, misses = _i64(), _i64(), _i64()
        tr = C.c_int32()
        _check(_L.kvcsim_pool_admit(self.h, kp, len(k), skip_begin, skip_end,
                                    ev.ctypes.data_as(_i64p), cap, C.byref(n_ev), C.byref(hits),
                                    C.byref(misses), C.byref(tr)))
        return {"evicted": ev[:n_ev.value].tolist(), "hits": hits.value, "misses": misses.value,
                "truncated": bool(tr.value)}

    def insert_replicated(self, blocks, chain_offset: int = 0) -> list:
        k, kp = _keys(blocks)
        cap = len(k) + self.size() + 1
        ev = np.zeros(cap, dtype=np.int64)
        n_ev = _i64()
        _check(_L.kvcsim_pool_insert_replicated(self.h, kp, len(k), chain_offset,
                                                ev.ctypes.data_as(_i64p), cap, C.byref(n_ev)))
        return ev[:n_ev.value].tolist()

    def match_prefix(self, blocks) -> int:
        k, kp = _keys(blocks)
        out = _i64()
        _check(_L.kvcsim_pool_match_prefix(self.h, kp, len(k), C.byref(out)))
        return out.value

    def contains(self, block) -> bool:
        out = C.c_int32()
        _check(_L.kvcsim_pool_contains(self.h, int(block), C.byref(out)))
        return bool(out.value)

    def size(self) -> int:
        return int(_L.kvcsim_pool_size(self.h))

    def stats(self):
        h, m = C.c_uint64(), C.c_uint64()
        _L.kvcsim_pool_stats(self.h, C.byref(h), C.byref(m))
        return int(h.value), int(m.value)


def match_prefix(pool: CachePool, blocks) -> int:
    return pool.match_prefix(blocks)


def find_best_prefix_match_batch(pools: Sequence[CachePool], ids: Sequence[int], keys,
                                 key_off, want_lens: bool = False):
    n_inst = len(pools)
    arr = (_vp * max(n_inst, 1))(*[p.h for p in pools])
    i = np.ascontiguousarray(ids, dtype=np.int32)
    k = np.ascontiguousarray(keys, dtype=np.int64)
    ko = np.ascontiguousarray(key_off, dtype=np.int64)
    n_req = len(ko) - 1
    lens = np.zeros(max(n_req * n_inst, 1), dtype=np.int64) if want_lens else None
    bl = np.zeros(max(n_req, 1), dtype=np.int64)
    bi = np.zeros(max(n_req, 1), dtype=np.int32)
    _check(_L.kvcsim_find_best_prefix_match_batch(
        arr, i.ctypes.data_as(_i32p), n_inst, k.ctypes.data_as(_i64p), ko.ctypes.data_as(_i64p),
        n_req, lens.ctypes.data_as(_i64p) if want_lens else None, bl.ctypes.data_as(_i64p),
        bi.ctypes.data_as(_i32p)))
    return (lens[: n_req * n_inst].reshape(n_req, n_inst) if want_lens else None,
            bl[:n_req], bi[:n_req])


def find_best_prefix_match(pools: Sequence[CachePool], ids: Sequence[int], keys):
    """Single-request form: (prefix_blocks, instance_id)."""
    _, bl, bi = find_best_prefix_match_batch(pools, ids, keys, [0, len(keys)])
    return int(bl[0]), int(bi[0])
