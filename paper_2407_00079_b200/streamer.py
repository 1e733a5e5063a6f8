"""Layer-wise KVCache streaming prefill -> decode (stages 2 -> 3 -> 4).

The engine is C++ in libkvx (``csrc/kvx_stream.cpp``, ``kvx_streamer_*`` in
include/kvx.h); this module is its Python face.

Reference behaviour made real: the prefill -> decode stream of a finished
prefill (proj/src/sim_engine.cpp:455-470; layer-wise launch/wait),
chunked-pipeline KV production (proj/src/perf_model.cpp:87-110), the
per-sender FIFO (proj/src/sim_engine.cpp:409-411).

Modes: ``local_fused`` / ``local_staged`` (N = 1), ``peer_fused`` /
``peer_ce`` / ``peer_pull`` (a prefill GPU and a decode GPU, one process each),
``peer_nccl`` (comparison: gather -> ncclSend / ncclRecv on the pair's own
communicator, in C++ too).
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import torch

from . import kvx
from .kvx import _L, _i64, _vp, check

MODES = {"local_fused": 0, "local_staged": 1, "peer_fused": 2, "peer_ce": 3, "peer_pull": 4,
         "peer_nccl": 5}
ROLES = {"local": 0, "sender": 1, "receiver": 2}


class KvxStreamerDesc(C.Structure):
    _fields_ = [("mode", C.c_int32), ("role", C.c_int32), ("ring", C.c_int32),
                ("time_launches", C.c_int32), ("slot_bytes", C.c_int64)]


def _sig(name, res, *args):
    f = getattr(_L, name)
    f.restype = res
    f.argtypes = list(args)


_sig("kvx_streamer_create", C.c_int, C.POINTER(KvxStreamerDesc), _vp, _vp, C.POINTER(_vp))
_sig("kvx_streamer_destroy", C.c_int, _vp)
_sig("kvx_streamer_export", C.c_int, _vp, _vp, _i64, C.POINTER(_i64))
_sig("kvx_streamer_connect", C.c_int, _vp, _vp, _i64, C.POINTER(kvx.KvxPoolDesc))
_sig("kvx_streamer_stream", _vp, _vp)
_sig("kvx_streamer_send", C.c_int, _vp, _vp, _vp, _i64, _i64, C.c_int32, C.c_int32, C.c_int32)
_sig("kvx_streamer_recv", C.c_int, _vp, _vp, _vp, _i64, _i64, C.c_int32, C.c_int32, C.c_int32)
_sig("kvx_streamer_finish", C.c_int, _vp, _vp)
_sig("kvx_streamer_after", C.c_int, _vp, _vp)
_sig("kvx_streamer_set_timing", C.c_int, _vp, C.c_int, C.c_int)
_sig("kvx_streamer_launch_stats", C.c_int, _vp, C.POINTER(_i64), C.POINTER(C.c_double),
     C.POINTER(C.c_double), C.c_int)
_sig("kvx_streamer_units", C.c_uint64, _vp)
_sig("kvx_streamer_check", C.c_int, _vp)
_sig("kvx_streamer_same_gpu", C.c_int, _vp)
_sig("kvx_streamer_set_pull_wait", C.c_int, _vp, C.c_int)
PULL_WAIT = {"gate": 0, "inline": 1, "stream": 2}
_sig("kvx_streamer_record_begin", C.c_int, _vp)
_sig("kvx_streamer_record_end", C.c_int, _vp)
_sig("kvx_streamer_replay", C.c_int, _vp)


class Streamer:
    """One end (or both, locally) of a prefill -> decode KV stream."""

    def __init__(self, mode: str, role: str, src: Optional[kvx.KVPool] = None,
                 dst: Optional[kvx.KVPool] = None, ring: int = 3, slot_bytes: int = 0,
                 time_launches: bool = False):
        self.mode, self.role = mode, role
        self.src, self.dst = src, dst
        d = KvxStreamerDesc(MODES[mode], ROLES[role], ring, int(time_launches), slot_bytes)
        h = _vp()
        check(_L.kvx_streamer_create(C.byref(d), src.h if src else None,
                                     dst.h if dst else None, C.byref(h)))
        self.h = h
        self.device = (src or dst).device
        self.stream = torch.cuda.ExternalStream(int(_L.kvx_streamer_stream(h)),
                                                device=self.device)

    def close(self):
        if getattr(self, "h", None) and kvx.alive():
            _L.kvx_streamer_destroy(self.h)
            self.h = None

    __del__ = close

    def export(self) -> bytes:
        n = _i64()
        check(_L.kvx_streamer_export(self.h, None, 0, C.byref(n)))
        buf = (C.c_uint8 * n.value)()
        check(_L.kvx_streamer_export(self.h, buf, n.value, C.byref(n)))
        return bytes(buf)

    def connect(self, blob: bytes, peer_pool: Optional[dict] = None):
        b = (C.c_uint8 * len(blob))(*blob)
        pd = None
        if peer_pool is not None:
            pd = kvx.KvxPoolDesc(peer_pool["layers"], peer_pool["block_size"],
                                 peer_pool["heads"], peer_pool["head_dim"],
                                 peer_pool["dtype_bytes"], peer_pool["slots"], self.device)
        check(_L.kvx_streamer_connect(self.h, b, len(blob), C.byref(pd) if pd else None))

    def send(self, src_table: torch.Tensor, dst_table: Optional[torch.Tensor], layer_lo: int,
             layer_hi: int, chunk_blocks: int = 0, layers_per_chunk: int = 1):
        n = src_table.numel()
        check(_L.kvx_streamer_send(self.h, src_table.data_ptr(),
                                   dst_table.data_ptr() if dst_table is not None else None, n,
                                   chunk_blocks or max(n, 1), layer_lo, layer_hi,
                                   layers_per_chunk))

    def recv(self, dst_table: torch.Tensor, layer_lo: int, layer_hi: int, chunk_blocks: int = 0,
             layers_per_chunk: int = 1, src_table: Optional[torch.Tensor] = None):
        n = dst_table.numel()
        check(_L.kvx_streamer_recv(self.h, src_table.data_ptr() if src_table is not None else None,
                                   dst_table.data_ptr(), n, chunk_blocks or max(n, 1), layer_lo,
                                   layer_hi, layers_per_chunk))

    def finish(self, stream=None):
        check(_L.kvx_streamer_finish(self.h, kvx._stream(stream) if stream is not None else None))

    def after(self, stream):
        check(_L.kvx_streamer_after(self.h, kvx._stream(stream)))

    def set_timing(self, on: bool, stride: int = 1):
        check(_L.kvx_streamer_set_timing(self.h, int(on), stride))

    def launch_stats(self, reset: bool = True):
        n, ms, b = _i64(), C.c_double(), C.c_double()
        check(_L.kvx_streamer_launch_stats(self.h, C.byref(n), C.byref(ms), C.byref(b),
                                           int(reset)))
        return {"launches": n.value, "avg_ms": ms.value, "avg_algorithmic_bytes": b.value}

    @property
    def units(self) -> int:
        return int(_L.kvx_streamer_units(self.h))

    def check(self):
        """Host-blocking: raise if a unit failed since the last check (a pulled
        unit that timed out waiting for the sender, or out-of-range table
        entries).  Call after finish() before using the decode slots."""
        check(_L.kvx_streamer_check(self.h))

    def set_pull_wait(self, mode: str):
        """PEER_PULL receiver: 'gate' (default), 'inline' or 'stream' (see kvx.h)."""
        check(_L.kvx_streamer_set_pull_wait(self.h, PULL_WAIT[mode]))

    @property
    def same_gpu(self) -> bool:
        """The connected peer process shares this GPU (waits are stream ops only)."""
        return bool(_L.kvx_streamer_same_gpu(self.h))

    def record_begin(self):
        """Capture the following sends (local fused mode) into a CUDA graph."""
        check(_L.kvx_streamer_record_begin(self.h))

    def record_end(self):
        check(_L.kvx_streamer_record_end(self.h))

    def replay(self):
        """Run the recorded step again: one cudaGraphLaunch."""
        check(_L.kvx_streamer_replay(self.h))
