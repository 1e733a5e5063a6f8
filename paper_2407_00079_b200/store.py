"""KVCache store of one instance (pool + index + slot allocator) and the
migration data path between instances -- Python face of ``kvx_store_*``
(include/kvx.h).  Reference: the Conductor's hot-spot migration
(proj/src/conductor.cpp:254-260) executed by the engine
(proj/src/sim_engine.cpp:399-419, abort at :605-639, landing at :641-650).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import kvx
from .kvx import _L, _i64, _vp, check

_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)


def _sig(name, res, *args):
    f = getattr(_L, name)
    f.restype = res
    f.argtypes = list(args)


_sig("kvx_store_create", C.c_int, C.POINTER(kvx.KvxPoolDesc), C.POINTER(_vp))
_sig("kvx_store_destroy", C.c_int, _vp)
_sig("kvx_store_pool", _vp, _vp)
_sig("kvx_store_index", _vp, _vp)
_sig("kvx_store_stream", _vp, _vp)
_sig("kvx_store_put", C.c_int, _vp, _i64p, _i64, _i32p)
_sig("kvx_store_get", C.c_int, _vp, _i64p, _i64, _i32p)
_sig("kvx_store_evict", C.c_int, _vp, _i64p, _i64)
_sig("kvx_store_migrate", C.c_int, _vp, _vp, _i64p, _i64, C.POINTER(_i64))
_sig("kvx_store_migrate_submit", C.c_int, _vp, _vp, _i64p, _i64, _vp, C.POINTER(C.c_uint64))
_sig("kvx_store_migrate_query", C.c_int, _vp, C.c_uint64)
_sig("kvx_store_migrate_wait", C.c_int, _vp, C.c_uint64, C.POINTER(_i64))
_sig("kvx_store_migrate_progress", C.c_int, _vp)


class KVStore:
    def __init__(self, layers: int, block_size: int, heads: int, head_dim: int,
                 dtype_bytes: int, slots: int, device: int = 0):
        self.desc = kvx.KvxPoolDesc(layers, block_size, heads, head_dim, dtype_bytes, slots,
                                    device)
        h = _vp()
        check(_L.kvx_store_create(C.byref(self.desc), C.byref(h)))
        self.h = h
        self.device = device
        self.layers, self.slots = layers, slots
        # non-owning view of the store's pool (for fill / verify / tests)
        self.pool = kvx.KVPool.__new__(kvx.KVPool)
        p = self.pool
        p.h = _vp(_L.kvx_store_pool(h))
        p.desc, p.layers, p.block_size, p.slots, p.device = self.desc, layers, block_size, slots, device
        p.slab = int(_L.kvx_pool_slab_bytes(p.h))
        p.nbytes = int(_L.kvx_pool_bytes(p.h))
        p.base = int(_L.kvx_pool_base(p.h))
        p.owned = False  # the store owns the pool

    def close(self):
        if getattr(self, "h", None) and kvx.alive():
            _L.kvx_store_destroy(self.h)
            self.h = None

    __del__ = close

    def put(self, keys) -> np.ndarray:
        k = np.ascontiguousarray(keys, dtype=np.int64)
        out = np.empty(max(len(k), 1), dtype=np.int32)
        check(_L.kvx_store_put(self.h, k.ctypes.data_as(_i64p), len(k), out.ctypes.data_as(_i32p)))
        return out[: len(k)]

    def get(self, keys) -> np.ndarray:
        k = np.ascontiguousarray(keys, dtype=np.int64)
        out = np.empty(max(len(k), 1), dtype=np.int32)
        check(_L.kvx_store_get(self.h, k.ctypes.data_as(_i64p), len(k), out.ctypes.data_as(_i32p)))
        return out[: len(k)]

    def evict(self, keys) -> None:
        k = np.ascontiguousarray(keys, dtype=np.int64)
        check(_L.kvx_store_evict(self.h, k.ctypes.data_as(_i64p), len(k)))

    def migrate_to(self, dst: "KVStore", keys) -> int:
        """Replicate `keys` (all must be resident here) into dst; returns the
        number of blocks copied.  Raises TransferAborted if any is missing."""
        k = np.ascontiguousarray(keys, dtype=np.int64)
        n = _i64()
        check(_L.kvx_store_migrate(self.h, dst.h, k.ctypes.data_as(_i64p), len(k), C.byref(n)))
        return n.value

    def migrate_submit(self, dst: "KVStore", keys, after_stream=None) -> int:
        """Queue a migration of `keys` to dst on this store's sender FIFO;
        returns a ticket.  It begins (residency check, copy launch) when the
        earlier migrations of this sender are done (sim_engine.cpp:409-411)."""
        k = np.ascontiguousarray(keys, dtype=np.int64)
        t = C.c_uint64()
        check(_L.kvx_store_migrate_submit(
            self.h, dst.h, k.ctypes.data_as(_i64p), len(k),
            kvx._stream(after_stream) if after_stream is not None else None, C.byref(t)))
        return t.value

    def migrate_query(self, ticket: int) -> str:
        """'done' | 'pending' | 'aborted' (never blocks)."""
        rc = _L.kvx_store_migrate_query(self.h, ticket)
        if rc == kvx.KVX_EAGAIN:
            return "pending"
        if rc == kvx.KVX_EABORTED:
            return "aborted"
        check(rc)
        return "done"

    def migrate_wait(self, ticket: int) -> int:
        """Block until the migration is done; returns the blocks that landed.
        Raises TransferAborted if the source evicted part of the range before
        the migration began."""
        n = _i64()
        check(_L.kvx_store_migrate_wait(self.h, ticket, C.byref(n)))
        return n.value

    def migrate_progress(self) -> None:
        check(_L.kvx_store_migrate_progress(self.h))
