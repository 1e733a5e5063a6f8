"""Python mirror of the KVCache hot-path interface over libkvx.so (C ABI).

The names follow the reference's plugin surface (kvcsim, /root/reference):

=====================  ==================================================
this module            reference interface it mirrors
=====================  ==================================================
``chain_hash``         ``kvcsim::chain_hash`` (proj/src/kvcache.cpp:14-23)
``chain_hash_batch``   batched prefix hashing (PAPER.md:290 PrefixHash)
``BlockIndex``         residency of ``CachePool`` (kvcache.hpp:44-102)
``match_prefix_batch`` ``CachePool::match_prefix`` + ``find_best_prefix_match``
                       (kvcache.cpp:150-158, conductor.cpp:57-73)
``KVPool.gather`` /    the KV bytes behind the reference's transfer model
``scatter`` /          (perf_model.cpp:51-59; sim_engine.cpp:399-419,455-476)
``copy_to``
``TransferEngine``     the Messenger's submit/wait with the per-sender FIFO
                       (sim_engine.cpp:409-411)
=====================  ==================================================

Errors: ``ValidationError`` (a ``ValueError``) for KVX_EINVAL -- the
reference's ``kvcsim::ValidationError`` -- and ``KvxError`` for CUDA failures.
There is no CPU fallback: importing this module without the compiled
``libkvx.so`` raises ``ImportError``; a call without a GPU raises ``KvxError``.
Device arrays are ``torch`` CUDA tensors (torch is plumbing only: memory,
streams); all compute runs in libkvx's sm_100a kernels.
"""
from __future__ import annotations

import atexit
import ctypes as C
import os
from typing import Optional, Sequence

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libkvx.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `make -C {_HERE}/csrc` or "
        "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")

_L = C.CDLL(LIB_PATH)

# Handles are released by __del__; at interpreter exit module globals are torn
# down in arbitrary order, so releases after exit starts are skipped (the
# process exit frees the device memory anyway).
_ALIVE = True


def _mark_exit():
    global _ALIVE
    _ALIVE = False


atexit.register(_mark_exit)


def alive() -> bool:
    return _ALIVE is True

KVX_OK, KVX_EINVAL, KVX_ENOMEM, KVX_ECUDA, KVX_EABORTED, KVX_EAGAIN = range(6)
KEY_EMPTY = -(1 << 63)
KEY_TOMBSTONE = -(1 << 63) + 1
MAX_INSTANCES = 64

_vp = C.c_void_p
_i64 = C.c_int64
_i32 = C.c_int32


def _sig(name, res, *args):
    f = getattr(_L, name)
    f.restype = res
    f.argtypes = list(args)
    return f


class KvxPoolDesc(C.Structure):
    _fields_ = [("layers", C.c_int32), ("block_size", C.c_int32), ("heads", C.c_int32),
                ("head_dim", C.c_int32), ("dtype_bytes", C.c_int32), ("slots", C.c_int64),
                ("device", C.c_int32)]


_sig("kvx_abi_version", C.c_int)
_sig("kvx_last_error", C.c_char_p)
_sig("kvx_launch_count", C.c_uint64)
_sig("kvx_sync", C.c_int, _vp)
_sig("kvx_chain_hash", _i64, _i64, C.c_uint64)
_sig("kvx_chain_hash_batch", C.c_int, _vp, _vp, _i64, _i64, _vp, _vp, _vp)
_sig("kvx_key_offsets", C.c_int, _vp, _i64, _i64, _vp, _vp)
_sig("kvx_hash_match_batch", C.c_int, _vp, _vp, _i64, _i64, _vp, _vp, C.POINTER(_vp),
     C.POINTER(_i32), _i64, _vp, _vp, _vp, _vp)
_sig("kvx_hash_match_check", C.c_int, _vp)
_sig("kvx_xmatch_key_buffer", C.c_int, _vp, _i64, C.POINTER(_vp))
_sig("kvx_xmatch_share_keys", C.c_int, _vp, _i64, _i64, _vp)
_sig("kvx_xmatch_hash_match", C.c_int, _vp, _vp, _vp, C.POINTER(_i64), _i64, _vp, _i64,
     C.POINTER(_vp), C.POINTER(_i32), _i64, _vp, _vp, C.POINTER(_vp), _vp)
_sig("kvx_index_create", C.c_int, C.c_int, _i64, C.POINTER(_vp))
_sig("kvx_index_destroy", C.c_int, _vp)
_sig("kvx_index_device", C.c_int, _vp)
_sig("kvx_index_insert", C.c_int, _vp, _vp, _vp, _i64, _vp)
_sig("kvx_index_erase", C.c_int, _vp, _vp, _i64, _vp)
_sig("kvx_index_lookup", C.c_int, _vp, _vp, _i64, _vp, _vp)
_sig("kvx_index_clear", C.c_int, _vp, _vp)
_sig("kvx_index_l2_pin", C.c_int, _vp, _vp, C.c_int)
_sig("kvx_index_reserve", C.c_int, _vp, _i64, _vp)
_sig("kvx_index_stats", C.c_int, _vp, C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_i64),
     C.POINTER(_i64), _vp)
_sig("kvx_match_prefix_batch", C.c_int, C.POINTER(_vp), C.POINTER(_i32), _i64, _vp, _vp, _i64,
     _vp, _vp, _vp, _vp)
_sig("kvx_match_prefix_packed", C.c_int, C.POINTER(_vp), C.POINTER(_i32), _i64, _vp, _vp, _i64,
     _vp, _vp)
_sig("kvx_best_unpack", C.c_int, _vp, _i64, _vp, _vp, _vp)
_sig("kvx_xmatch_create", C.c_int, C.c_int, C.c_int, C.c_int, _i64, C.POINTER(_vp))
_sig("kvx_xmatch_destroy", C.c_int, _vp)
_sig("kvx_xmatch_export", C.c_int, _vp, C.c_char_p, _i64, C.POINTER(_i64))
_sig("kvx_xmatch_connect", C.c_int, _vp, C.c_char_p, _i64)
_sig("kvx_xmatch_run", C.c_int, _vp, C.POINTER(_vp), C.POINTER(_i32), _i64, _vp, _vp, _i64, _vp,
     _vp, _vp)
_sig("kvx_pool_create", C.c_int, C.POINTER(KvxPoolDesc), C.POINTER(_vp))
_sig("kvx_pool_create_view", C.c_int, C.POINTER(KvxPoolDesc), _vp, C.POINTER(_vp))
_sig("kvx_pool_create_host", C.c_int, C.POINTER(KvxPoolDesc), C.POINTER(_vp))
_sig("kvx_pool_is_host", C.c_int, _vp)
_sig("kvx_layer_io_create", C.c_int, C.c_int, C.c_int32, C.POINTER(_vp))
_sig("kvx_layer_io_destroy", C.c_int, _vp)
_sig("kvx_layer_io_load_stream", _vp, _vp)
_sig("kvx_layer_io_store_stream", _vp, _vp)
_sig("kvx_layer_load_launch", C.c_int, _vp, _vp, _vp, _vp, _vp, _i64, _i32, _i32, _vp)
_sig("kvx_layer_load_wait", C.c_int, _vp, _i32, _vp)
_sig("kvx_layer_store_launch", C.c_int, _vp, _vp, _vp, _vp, _vp, _i64, _i32, _i32, _vp)
_sig("kvx_layer_store_wait_all", C.c_int, _vp, _vp)
_sig("kvx_layer_load_range", C.c_int, _vp, _vp, _i64, _vp, _i64, _i64, _i32, _i32, _vp)
_sig("kvx_layer_store_range", C.c_int, _vp, _vp, _i64, _vp, _i64, _i64, _i32, _i32, _vp)
_sig("kvx_pool_destroy", C.c_int, _vp)
_sig("kvx_pool_base", _vp, _vp)
_sig("kvx_pool_slab_bytes", _i64, _vp)
_sig("kvx_pool_bytes", _i64, _vp)
_sig("kvx_pool_fill_synthetic", C.c_int, _vp, C.c_uint32, _vp)
_sig("kvx_pool_verify", C.c_int, _vp, _vp, C.c_uint32, _vp, _i64, _i32, _i32, _vp, _vp)
_sig("kvx_gather", C.c_int, _vp, _vp, _i64, _i32, _i32, _vp, _vp)
_sig("kvx_scatter", C.c_int, _vp, _vp, _i64, _i32, _i32, _vp, _vp)
_sig("kvx_copy_paged", C.c_int, _vp, _vp, _vp, _vp, _i64, _i32, _i32, _vp)
_sig("kvx_set_copy_impl", C.c_int, C.c_int)
_sig("kvx_copy_check", C.c_int, _vp)
_sig("kvx_xfer_create", C.c_int, C.c_int, C.POINTER(_vp))
_sig("kvx_xfer_destroy", C.c_int, _vp)
_sig("kvx_xfer_stream", _vp, _vp)
_sig("kvx_transfer_submit", C.c_int, _vp, _vp, _vp, _i64, _vp, C.POINTER(C.c_uint64))
_sig("kvx_transfer_wait", C.c_int, _vp, C.c_uint64)
_sig("kvx_transfer_wait_stream", C.c_int, _vp, C.c_uint64, _vp)
_sig("kvx_transfer_query", C.c_int, _vp, C.c_uint64)
_sig("kvx_transfer_signal", C.c_int, _vp, _vp, C.c_uint64)
_sig("kvx_ipc_export", C.c_int, _vp, C.POINTER(C.c_uint8))
_sig("kvx_ipc_open", C.c_int, C.POINTER(C.c_uint8), C.c_int, C.POINTER(_vp))
_sig("kvx_ipc_close", C.c_int, _vp)
_sig("kvx_enable_peer", C.c_int, C.c_int, C.c_int)
_sig("kvx_signal_write", C.c_int, _vp, _vp, C.c_uint64)
_sig("kvx_signal_wait", C.c_int, _vp, _vp, C.c_uint64)
_sig("kvx_device_alloc", C.c_int, C.c_int, _i64, C.POINTER(_vp))
_sig("kvx_device_free", C.c_int, C.c_int, _vp)
_sig("kvx_slot_alloc_create", C.c_int, _i64, C.POINTER(_vp))
_sig("kvx_slot_alloc_destroy", C.c_int, _vp)
_sig("kvx_slot_alloc_free_count", _i64, _vp)
_sig("kvx_slot_alloc_take", C.c_int, _vp, _i64, C.POINTER(_i32))
_sig("kvx_slot_alloc_mark", C.c_int, _vp, C.POINTER(_i32), _i64)
_sig("kvx_slot_alloc_release", C.c_int, _vp, C.POINTER(_i32), _i64)


class KvxError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"kvx status {status}: {msg}")
        self.status = status


class ValidationError(ValueError):
    """KVX_EINVAL: the reference's kvcsim::ValidationError (errors.hpp:18-21)."""


class TransferAborted(KvxError):
    """KVX_EABORTED: the transfer source evicted the range (sim_engine.cpp:605-639)."""


def check(status: int) -> int:
    if status in (KVX_OK, KVX_EAGAIN):
        return status
    msg = (_L.kvx_last_error() or b"").decode(errors="replace")
    if status == KVX_EINVAL:
        raise ValidationError(msg)
    if status == KVX_EABORTED:
        raise TransferAborted(status, msg)
    raise KvxError(status, msg)


def abi_version() -> int:
    return int(_L.kvx_abi_version())


def launch_count() -> int:
    """Kernels launched by libkvx in this process (bench's gpu_launches)."""
    return int(_L.kvx_launch_count())


def _stream(stream=None) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _torch_stream(stream, device) -> torch.cuda.Stream:
    if stream is None:
        return torch.cuda.current_stream(device)
    if isinstance(stream, int):
        return torch.cuda.ExternalStream(stream, device=device)
    return stream


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    assert t.is_cuda and t.is_contiguous(), "device arrays must be contiguous CUDA tensors"
    return t.data_ptr()


def set_copy_impl(impl: str) -> None:
    """'lsu' (128-bit loads/stores) or 'tma' (cp.async.bulk pipeline)."""
    check(_L.kvx_set_copy_impl({"lsu": 0, "tma": 1}[impl]))


def copy_check(stream=None) -> None:
    """Raise ValidationError (KVX_EINVAL) if a gather / scatter / paged copy met a block
    table entry outside [0, slots) since the last check on the current device
    (that block was skipped, not copied).  Synchronizes `stream`."""
    check(_L.kvx_copy_check(_stream(stream)))


# ---- stage 1a ---------------------------------------------------------------

def chain_hash(prev_key: int, content_hash: int) -> int:
    """Scalar kvcsim::chain_hash (bit-identical)."""
    return int(_L.kvx_chain_hash(int(prev_key), int(content_hash) & 0xFFFFFFFFFFFFFFFF))


def key_offsets(tok_off: torch.Tensor, bs: int, out: Optional[torch.Tensor] = None,
                stream=None) -> torch.Tensor:
    """Exclusive scan of ceil(len/bs) per request (kvx_key_offsets kernel)."""
    assert tok_off.dtype == torch.int64
    with torch.cuda.stream(_torch_stream(stream, tok_off.device)):
        if out is None:
            out = torch.empty(len(tok_off), dtype=torch.int64, device=tok_off.device)
    check(_L.kvx_key_offsets(_ptr(tok_off), len(tok_off) - 1, bs, _ptr(out), _stream(stream)))
    return out


def chain_hash_batch(tokens: torch.Tensor, tok_off: torch.Tensor, bs: int,
                     key_off: Optional[torch.Tensor] = None, keys: Optional[torch.Tensor] = None,
                     stream=None):
    """Prefix-chained block keys of a batch of requests (K1).  Returns
    (keys, key_off).  tokens int32, tok_off int64 (n_req+1), both on the GPU."""
    assert tokens.dtype == torch.int32 and tok_off.dtype == torch.int64
    # the offsets and the output are made on the stream the kernel runs on
    with torch.cuda.stream(_torch_stream(stream, tokens.device)):
        if key_off is None:
            key_off = key_offsets(tok_off, bs, stream=stream)
        if keys is None:
            n_keys = int(key_off[-1].item())
            keys = torch.empty(max(n_keys, 1), dtype=torch.int64, device=tokens.device)[:n_keys]
    check(_L.kvx_chain_hash_batch(_ptr(tokens) if tokens.numel() else None, _ptr(tok_off),
                                  len(tok_off) - 1, bs, _ptr(key_off),
                                  _ptr(keys) if keys.numel() else None, _stream(stream)))
    return keys, key_off


# ---- stage 1b -----------------------------------------------------------------

class BlockIndex:
    """GPU block index (int64 key -> int64 value), one per prefill instance."""

    def __init__(self, device: int = 0, capacity_hint: int = 1024):
        h = _vp()
        check(_L.kvx_index_create(device, capacity_hint, C.byref(h)))
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None) and _ALIVE is True:
            _L.kvx_index_destroy(self.h)
            self.h = None

    __del__ = close

    def insert(self, keys: torch.Tensor, values: Optional[torch.Tensor] = None, stream=None):
        if keys.numel():
            check(_L.kvx_index_insert(self.h, _ptr(keys), _ptr(values), keys.numel(),
                                      _stream(stream)))

    def erase(self, keys: torch.Tensor, stream=None):
        if keys.numel():
            check(_L.kvx_index_erase(self.h, _ptr(keys), keys.numel(), _stream(stream)))

    def lookup(self, keys: torch.Tensor, out: Optional[torch.Tensor] = None, stream=None):
        if out is None:
            out = torch.empty_like(keys)
        if keys.numel():
            check(_L.kvx_index_lookup(self.h, _ptr(keys), keys.numel(), _ptr(out),
                                      _stream(stream)))
        return out

    def clear(self, stream=None):
        check(_L.kvx_index_clear(self.h, _stream(stream)))

    def reserve(self, min_keys: int, stream=None):
        check(_L.kvx_index_reserve(self.h, min_keys, _stream(stream)))

    def l2_pin(self, stream, on: bool = True):
        """Keep the key table L2-resident for kernels on `stream` (persisting
        access-policy window)."""
        check(_L.kvx_index_l2_pin(self.h, _stream(stream), int(on)))

    def stats(self, stream=None):
        live, tomb, slots, rej = _i64(), _i64(), _i64(), _i64()
        check(_L.kvx_index_stats(self.h, C.byref(live), C.byref(tomb), C.byref(slots),
                                 C.byref(rej), _stream(stream)))
        return {"live": live.value, "tombstones": tomb.value, "slots": slots.value,
                "rejected": rej.value}


def match_prefix_batch(indices: Sequence[BlockIndex], inst_ids: Sequence[int], keys: torch.Tensor,
                       key_off: torch.Tensor, want_lens: bool = True, stream=None, out=None):
    """K2: per-(request, instance) match_prefix and the per-request
    find_best_prefix_match.  Returns (lens[n_req, n_inst] or None, best_len, best_id)."""
    n_inst = len(indices)
    n_req = len(key_off) - 1
    dev = keys.device
    arr = (_vp * max(n_inst, 1))(*[i.h for i in indices])
    ids = (_i32 * max(n_inst, 1))(*[int(i) for i in inst_ids])
    if out is None:
        lens = torch.empty((n_req, n_inst), dtype=torch.int64, device=dev) if want_lens else None
        best_len = torch.empty(n_req, dtype=torch.int64, device=dev)
        best_id = torch.empty(n_req, dtype=torch.int32, device=dev)
    else:
        lens, best_len, best_id = out
    check(_L.kvx_match_prefix_batch(arr, ids, n_inst, _ptr(keys) if keys.numel() else None,
                                    _ptr(key_off), n_req, _ptr(lens) if lens is not None else None,
                                    _ptr(best_len), _ptr(best_id), _stream(stream)))
    return lens, best_len, best_id


def hash_match_batch(tokens: torch.Tensor, tok_off: torch.Tensor, bs: int,
                     indices: Sequence["BlockIndex"], inst_ids: Sequence[int],
                     key_off: Optional[torch.Tensor] = None, keys: Optional[torch.Tensor] = None,
                     want_lens: bool = False, stream=None, out=None):
    """Stage 1 in one call (kvx_hash_match_batch): block keys of the batch and
    every request's match against the instances, the match of a request
    starting as soon as its keys are stored.  Returns (keys, key_off, lens or
    None, best_len, best_id)."""
    assert tokens.dtype == torch.int32 and tok_off.dtype == torch.int64
    n_inst = len(indices)
    n_req = len(tok_off) - 1
    dev = tokens.device
    with torch.cuda.stream(_torch_stream(stream, dev)):
        if key_off is None:
            key_off = key_offsets(tok_off, bs, stream=stream)
        if keys is None:
            n_keys = int(key_off[-1].item())
            keys = torch.empty(max(n_keys, 1), dtype=torch.int64, device=dev)[:n_keys]
        if out is None:
            lens = torch.empty((n_req, n_inst), dtype=torch.int64, device=dev) if want_lens else None
            best_len = torch.empty(n_req, dtype=torch.int64, device=dev)
            best_id = torch.empty(n_req, dtype=torch.int32, device=dev)
        else:
            lens, best_len, best_id = out
    arr = (_vp * max(n_inst, 1))(*[i.h for i in indices])
    ids = (_i32 * max(n_inst, 1))(*[int(i) for i in inst_ids])
    check(_L.kvx_hash_match_batch(_ptr(tokens) if tokens.numel() else None, _ptr(tok_off),
                                  n_req, bs, _ptr(key_off), _ptr(keys) if keys.numel() else None,
                                  arr, ids, n_inst, _ptr(lens) if lens is not None else None,
                                  _ptr(best_len), _ptr(best_id), _stream(stream)))
    return keys, key_off, lens, best_len, best_id


def hash_match_check(stream=None) -> None:
    """Host-blocking: raise if a fused stage-1 call lost a request (a defect)."""
    check(_L.kvx_hash_match_check(_stream(stream)))


def match_prefix_packed(indices: Sequence[BlockIndex], inst_ids: Sequence[int],
                        keys: torch.Tensor, key_off: torch.Tensor, out: Optional[torch.Tensor] = None,
                        stream=None) -> torch.Tensor:
    """Per request the packed best word (len << 32 | ~ordered(id)), an int64
    tensor whose element-wise MAX over GPUs (all-reduce) is the global
    find_best_prefix_match; decode with best_unpack."""
    n_inst = len(indices)
    n_req = len(key_off) - 1
    arr = (_vp * max(n_inst, 1))(*[i.h for i in indices])
    ids = (_i32 * max(n_inst, 1))(*[int(i) for i in inst_ids])
    if out is None:
        out = torch.empty(n_req, dtype=torch.int64, device=keys.device)
    check(_L.kvx_match_prefix_packed(arr, ids, n_inst, _ptr(keys) if keys.numel() else None,
                                     _ptr(key_off), n_req, _ptr(out), _stream(stream)))
    return out


class XMatch:
    """Cross-GPU find_best_prefix_match without a collective (kvx_xmatch_*):
    every rank's match kernel MAXes its packed words into every rank's result
    buffer over NVLink, stream-ordered flags close the step.  Create on every
    rank, exchange ``export()`` blobs, ``connect`` every blob (own included is
    a no-op), then call ``run`` on every rank once per batch."""

    def __init__(self, device: int, rank: int, world: int, max_req: int):
        h = _vp()
        check(_L.kvx_xmatch_create(device, rank, world, max_req, C.byref(h)))
        self.h, self.device, self.rank, self.world = h, device, rank, world

    def export(self) -> bytes:
        n = _i64()
        check(_L.kvx_xmatch_export(self.h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        check(_L.kvx_xmatch_export(self.h, buf, n.value, C.byref(n)))
        return buf.raw[: n.value]

    def connect(self, blob: bytes) -> None:
        check(_L.kvx_xmatch_connect(self.h, blob, len(blob)))

    def key_buffer(self, max_keys: int) -> torch.Tensor:
        """This rank's copy of the batch-wide key buffer (request-sharded
        hashing); call before export()."""
        p = _vp()
        check(_L.kvx_xmatch_key_buffer(self.h, max_keys, C.byref(p)))
        self.max_keys = max_keys
        # valid while this XMatch lives (no back reference: no cycle)
        return _wrap_device_bytes(int(p.value), 8 * max_keys, self.device).view(torch.int64)

    def share_keys(self, key_lo: int, key_hi: int, stream=None) -> None:
        """Push this rank's hashed shard [key_lo, key_hi) to every peer (copy
        engine over NVLink); `stream` then waits for every peer's shard."""
        check(_L.kvx_xmatch_share_keys(self.h, key_lo, key_hi, _stream(stream)))

    def hash_match(self, tokens: torch.Tensor, tok_off: torch.Tensor, bounds: Sequence[int],
                   bs: int, key_off: torch.Tensor, indices: Sequence[BlockIndex],
                   inst_ids: Sequence[int], out=None, stream=None):
        """Request-sharded stage 1 with the key exchange inside the match
        kernel: rank k hashes requests [bounds[k], bounds[k+1]) of the batch
        into its own key buffer; every rank's match kernel follows the keys
        of the WHOLE batch where they are produced (NVLink loads of the
        owner's buffer) against its instances and MAXes the result into every
        rank's buffer.  Collective, once per step, same bounds on every rank.
        Needs key_buffer() sized for the batch, bs % 16 == 0 and one GPU per
        rank.  Returns (best_len, best_id, keys) -- keys: this rank's buffer
        of the step (its own shard's keys valid; until the step after next)."""
        n_inst = len(indices)
        n_req = len(key_off) - 1
        arr = (_vp * max(n_inst, 1))(*[i.h for i in indices])
        ids = (_i32 * max(n_inst, 1))(*[int(i) for i in inst_ids])
        b = (_i64 * len(bounds))(*[int(v) for v in bounds])
        if out is None:
            out = (torch.empty(n_req, dtype=torch.int64, device=key_off.device),
                   torch.empty(n_req, dtype=torch.int32, device=key_off.device))
        best_len, best_id = out
        n_keys = int(key_off[-1].item())
        if n_keys > getattr(self, "max_keys", 0):
            raise ValidationError("XMatch.hash_match: the batch has more keys than key_buffer()")
        kp = _vp()
        check(_L.kvx_xmatch_hash_match(self.h, _ptr(tokens), _ptr(tok_off), b, bs, _ptr(key_off),
                                       n_req, arr, ids, n_inst, _ptr(best_len), _ptr(best_id),
                                       C.byref(kp), _stream(stream)))
        keys = (_wrap_device_bytes(int(kp.value), 8 * n_keys, self.device).view(torch.int64)
                if kp.value and n_keys else None)
        return best_len, best_id, keys

    def run(self, indices: Sequence[BlockIndex], inst_ids: Sequence[int], keys: torch.Tensor,
            key_off: torch.Tensor, out=None, stream=None):
        n_inst = len(indices)
        n_req = len(key_off) - 1
        arr = (_vp * max(n_inst, 1))(*[i.h for i in indices])
        ids = (_i32 * max(n_inst, 1))(*[int(i) for i in inst_ids])
        if out is None:
            out = (torch.empty(n_req, dtype=torch.int64, device=keys.device),
                   torch.empty(n_req, dtype=torch.int32, device=keys.device))
        best_len, best_id = out
        check(_L.kvx_xmatch_run(self.h, arr, ids, n_inst, _ptr(keys) if keys.numel() else None,
                                _ptr(key_off), n_req, _ptr(best_len), _ptr(best_id),
                                _stream(stream)))
        return best_len, best_id

    def __del__(self):
        if getattr(self, "h", None) and alive():
            _L.kvx_xmatch_destroy(self.h)
            self.h = None


def best_unpack(packed: torch.Tensor, stream=None):
    n = packed.numel()
    best_len = torch.empty(n, dtype=torch.int64, device=packed.device)
    best_id = torch.empty(n, dtype=torch.int32, device=packed.device)
    check(_L.kvx_best_unpack(_ptr(packed), n, _ptr(best_len), _ptr(best_id), _stream(stream)))
    return best_len, best_id


# ---- paged KV pool and stages 2/4 ---------------------------------------------

class KVPool:
    """Paged KV pool: HBM layout [layer][K|V][slot][block_size][heads][head_dim]."""

    def __init__(self, layers: int, block_size: int, heads: int, head_dim: int, dtype_bytes: int,
                 slots: int, device: int = 0, base_ptr: Optional[int] = None, host: bool = False):
        """host=True: the CPU-DRAM tier (pinned, device-mapped host memory, same
        layout), accessed by GPU `device`'s copy kernels over PCIe."""
        self.desc = KvxPoolDesc(layers, block_size, heads, head_dim, dtype_bytes, slots, device)
        h = _vp()
        self.host = host
        if host:
            check(_L.kvx_pool_create_host(C.byref(self.desc), C.byref(h)))
        elif base_ptr is None:
            check(_L.kvx_pool_create(C.byref(self.desc), C.byref(h)))
        else:
            check(_L.kvx_pool_create_view(C.byref(self.desc), _vp(base_ptr), C.byref(h)))
        self.h = h
        self.layers, self.block_size, self.slots, self.device = layers, block_size, slots, device
        self.slab = int(_L.kvx_pool_slab_bytes(h))
        self.nbytes = int(_L.kvx_pool_bytes(h))
        self.base = int(_L.kvx_pool_base(h))

    def close(self):
        if getattr(self, "h", None) and getattr(self, "owned", True) and _ALIVE is True:
            _L.kvx_pool_destroy(self.h)
            self.h = None

    __del__ = close

    def buffer_bytes(self, n_blocks: int, layer_lo: int, layer_hi: int) -> int:
        return (layer_hi - layer_lo) * 2 * n_blocks * self.slab

    def fill_synthetic(self, pool_id: int, stream=None):
        check(_L.kvx_pool_fill_synthetic(self.h, pool_id, _stream(stream)))

    def verify(self, dst_table: torch.Tensor, src_pool_id: int, src_table: torch.Tensor,
               layer_lo: int, layer_hi: int, counter: Optional[torch.Tensor] = None, stream=None):
        """Adds to `counter` (uint64 as int64 tensor[1]) the number of 64-bit words of
        this pool's dst slabs that differ from the synthetic source content."""
        if counter is None:
            counter = torch.zeros(1, dtype=torch.int64, device=f"cuda:{self.device}")
        check(_L.kvx_pool_verify(self.h, _ptr(dst_table), src_pool_id, _ptr(src_table),
                                 dst_table.numel(), layer_lo, layer_hi, _ptr(counter),
                                 _stream(stream)))
        return counter

    def gather(self, src_table: torch.Tensor, layer_lo: int, layer_hi: int, buf_ptr: int,
               stream=None):
        check(_L.kvx_gather(self.h, _ptr(src_table), src_table.numel(), layer_lo, layer_hi,
                            _vp(buf_ptr), _stream(stream)))

    def scatter(self, dst_table: torch.Tensor, layer_lo: int, layer_hi: int, buf_ptr: int,
                stream=None):
        check(_L.kvx_scatter(self.h, _ptr(dst_table), dst_table.numel(), layer_lo, layer_hi,
                             _vp(buf_ptr), _stream(stream)))

    def copy_to(self, dst: "KVPool", src_table: torch.Tensor, dst_table: torch.Tensor,
                layer_lo: int, layer_hi: int, stream=None):
        """Fused paged -> paged copy (dst may be a peer view)."""
        assert src_table.numel() == dst_table.numel()
        check(_L.kvx_copy_paged(self.h, _ptr(src_table), dst.h, _ptr(dst_table),
                                src_table.numel(), layer_lo, layer_hi, _stream(stream)))

    def host_array(self):
        """numpy uint8 view of a host (DRAM-tier) pool's bytes (no copy)."""
        import numpy as np
        assert self.host, "host_array: not a host pool"
        return np.ctypeslib.as_array((C.c_uint8 * self.nbytes).from_address(self.base))

    def tensor_view(self) -> torch.Tensor:
        """uint8 torch view of the whole pool (tests only; does not own memory)."""
        return _wrap_device_bytes(self.base, self.nbytes, self.device, owner=self)


def _wrap_device_bytes(ptr: int, nbytes: int, device: int, owner=None) -> torch.Tensor:
    class _CAI:
        def __init__(self):
            self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                             "data": (ptr, False), "version": 2, "strides": None}
    with torch.cuda.device(device):
        t = torch.as_tensor(_CAI(), device=f"cuda:{device}")
    t._kvx_owner = owner
    return t


# ---- stage 3 -----------------------------------------------------------------

class TransferEngine:
    """One in-order copy-engine queue per source GPU (the per-sender FIFO)."""

    def __init__(self, device: int = 0):
        h = _vp()
        check(_L.kvx_xfer_create(device, C.byref(h)))
        self.h = h
        self.device = device
        self.stream_handle = int(_L.kvx_xfer_stream(h))

    def close(self):
        if getattr(self, "h", None) and _ALIVE is True:
            _L.kvx_xfer_destroy(self.h)
            self.h = None

    __del__ = close

    def submit(self, dst_ptr: int, src_ptr: int, nbytes: int, after_stream=None) -> int:
        t = C.c_uint64()
        after = None if after_stream is None else _vp(_stream(after_stream))
        check(_L.kvx_transfer_submit(self.h, _vp(dst_ptr), _vp(src_ptr), nbytes, after,
                                     C.byref(t)))
        return t.value

    def wait(self, ticket: int) -> None:
        check(_L.kvx_transfer_wait(self.h, ticket))

    def wait_stream(self, ticket: int, stream=None) -> None:
        check(_L.kvx_transfer_wait_stream(self.h, ticket, _stream(stream)))

    def done(self, ticket: int) -> bool:
        return check(_L.kvx_transfer_query(self.h, ticket)) == KVX_OK

    def signal(self, flag_ptr: int, value: int) -> None:
        check(_L.kvx_transfer_signal(self.h, _vp(flag_ptr), value))


def ipc_export(ptr: int) -> bytes:
    buf = (C.c_uint8 * 64)()
    check(_L.kvx_ipc_export(_vp(ptr), buf))
    return bytes(buf)


def ipc_open(handle: bytes, device: int) -> int:
    buf = (C.c_uint8 * 64)(*handle)
    p = _vp()
    check(_L.kvx_ipc_open(buf, device, C.byref(p)))
    return int(p.value)


def ipc_close(ptr: int) -> None:
    check(_L.kvx_ipc_close(_vp(ptr)))


def enable_peer(device: int, peer: int) -> None:
    check(_L.kvx_enable_peer(device, peer))


def signal_write(flag_ptr: int, value: int, stream=None) -> None:
    check(_L.kvx_signal_write(_vp(_stream(stream)), _vp(flag_ptr), value))


def signal_wait(flag_ptr: int, value: int, stream=None) -> None:
    check(_L.kvx_signal_wait(_vp(_stream(stream)), _vp(flag_ptr), value))


class LayerIO:
    """Layer-wise DRAM <-> HBM KV load / store with launch / wait per layer
    (the reference's cache_load_time / layerwise_effective_prefill,
    proj/src/perf_model.cpp:73-85)."""

    def __init__(self, device: int, max_layers: int):
        h = _vp()
        check(_L.kvx_layer_io_create(device, max_layers, C.byref(h)))
        self.h, self.device = h, device
        self.load_stream = torch.cuda.ExternalStream(int(_L.kvx_layer_io_load_stream(h)),
                                                     device=device)
        self.store_stream = torch.cuda.ExternalStream(int(_L.kvx_layer_io_store_stream(h)),
                                                      device=device)

    def close(self):
        if getattr(self, "h", None) and _ALIVE is True:
            _L.kvx_layer_io_destroy(self.h)
            self.h = None

    __del__ = close

    def load(self, host: "KVPool", host_table: torch.Tensor, dev: "KVPool",
             dev_table: torch.Tensor, layer_lo: int, layer_hi: int, after=None):
        assert host_table.numel() == dev_table.numel()
        check(_L.kvx_layer_load_launch(self.h, host.h, _ptr(host_table), dev.h, _ptr(dev_table),
                                       dev_table.numel(), layer_lo, layer_hi,
                                       _stream(after) if after is not None else None))

    def wait_layer(self, layer: int, stream=None):
        check(_L.kvx_layer_load_wait(self.h, layer, _stream(stream)))

    def store(self, dev: "KVPool", dev_table: torch.Tensor, host: "KVPool",
              host_table: torch.Tensor, layer_lo: int, layer_hi: int, after=None):
        assert host_table.numel() == dev_table.numel()
        check(_L.kvx_layer_store_launch(self.h, dev.h, _ptr(dev_table), host.h, _ptr(host_table),
                                        dev_table.numel(), layer_lo, layer_hi,
                                        _stream(after) if after is not None else None))

    def load_range(self, host: "KVPool", host_first: int, dev: "KVPool", dev_first: int, n: int,
                   layer_lo: int, layer_hi: int, after=None):
        """Contiguous runs: two copy-engine copies per layer, no kernel."""
        check(_L.kvx_layer_load_range(self.h, host.h, host_first, dev.h, dev_first, n, layer_lo,
                                      layer_hi, _stream(after) if after is not None else None))

    def store_range(self, dev: "KVPool", dev_first: int, host: "KVPool", host_first: int, n: int,
                    layer_lo: int, layer_hi: int, after=None):
        check(_L.kvx_layer_store_range(self.h, dev.h, dev_first, host.h, host_first, n, layer_lo,
                                       layer_hi, _stream(after) if after is not None else None))

    def wait_stores(self, stream=None):
        """stream None: host-blocking."""
        check(_L.kvx_layer_store_wait_all(self.h, _stream(stream) if stream is not None
                                          else None))


class DeviceBuffer:
    """Raw cudaMalloc'd bytes (IPC-exportable), optionally viewed as a tensor."""

    def __init__(self, nbytes: int, device: int = 0):
        p = _vp()
        check(_L.kvx_device_alloc(device, nbytes, C.byref(p)))
        self.ptr = int(p.value)
        self.nbytes = nbytes
        self.device = device

    def close(self):
        if getattr(self, "ptr", 0) and _ALIVE is True:
            _L.kvx_device_free(self.device, _vp(self.ptr))
            self.ptr = 0

    __del__ = close

    def tensor(self, dtype=torch.uint8) -> torch.Tensor:
        t = _wrap_device_bytes(self.ptr, self.nbytes, self.device, owner=self)
        return t.view(dtype)


class SlotAllocator:
    """Decode-side block table allocator: n lowest free slots, ascending."""

    def __init__(self, slots: int):
        h = _vp()
        check(_L.kvx_slot_alloc_create(slots, C.byref(h)))
        self.h = h
        self.slots = slots

    def close(self):
        if getattr(self, "h", None) and _ALIVE is True:
            _L.kvx_slot_alloc_destroy(self.h)
            self.h = None

    __del__ = close

    @property
    def free(self) -> int:
        return int(_L.kvx_slot_alloc_free_count(self.h))

    def take(self, n: int, out=None):
        import numpy as np
        if out is None:
            out = np.empty(max(n, 1), dtype=np.int32)
        check(_L.kvx_slot_alloc_take(self.h, n, out.ctypes.data_as(C.POINTER(_i32))))
        return out[:n]

    def mark(self, slots) -> None:
        import numpy as np
        a = np.ascontiguousarray(slots, dtype=np.int32)
        check(_L.kvx_slot_alloc_mark(self.h, a.ctypes.data_as(C.POINTER(_i32)), len(a)))

    def release(self, slots) -> None:
        import numpy as np
        a = np.ascontiguousarray(slots, dtype=np.int32)
        check(_L.kvx_slot_alloc_release(self.h, a.ctypes.data_as(C.POINTER(_i32)), len(a)))


def sync(stream=None) -> None:
    check(_L.kvx_sync(_vp(_stream(stream))))
