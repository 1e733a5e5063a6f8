"""Batched Conductor scoring -- the kvcache-centric schedule() of the
reference (proj/src/conductor.cpp:126-262) for a whole batch of requests
against one cluster snapshot, on the GPU (``kvx_schedule_batch``).

Typical use: ``lens, _, _ = match_prefix_batch(indices, ids, keys, key_off)``
then ``schedule_batch(perf, slo, prefill, decode, input_len, lens)``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import kvx
from .kvx import _L, _i64, _vp, check

PREFILL_DT = np.dtype([("id", "<i4"), ("pad", "<i4"), ("busy_until_ms", "<f8"),
                       ("sender_busy_until_ms", "<f8"), ("queued_work_ms", "<f8")], align=True)
DECODE_DT = np.dtype([("id", "<i4"), ("pad", "<i4"), ("batch_size", "<i8"),
                      ("resident_kv_tokens", "<i8")], align=True)
DECISION_DT = np.dtype([("accepted", "<i4"), ("reject_reason", "<i4"), ("prefill_id", "<i4"),
                        ("decode_id", "<i4"), ("local_prefix_blocks", "<i8"),
                        ("used_prefix_blocks", "<i8"), ("best_prefix_blocks", "<i8"),
                        ("best_instance_id", "<i4"), ("migrate", "<i4"),
                        ("migrate_source", "<i4"), ("pad", "<i4"),
                        ("migrate_prefix_blocks", "<i8"), ("queue_ms", "<f8"),
                        ("transfer_ms", "<f8"), ("exec_ms", "<f8"), ("ttft_ms", "<f8"),
                        ("tbt_ms", "<f8")], align=True)


class KvxPerfParams(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("alpha_mlp", "beta_attn", "gamma_decode",
                                          "delta_decode", "epsilon_decode",
                                          "kv_bytes_per_token", "link_bandwidth",
                                          "load_bandwidth")] + \
               [("prefill_chunk", C.c_int64), ("cpp_group_size", C.c_int64)]


class KvxSchedParams(C.Structure):
    _fields_ = [("l_ttft_ms", C.c_double), ("l_tbt_ms", C.c_double),
                ("kvcache_balancing_threshold", C.c_double), ("now_ms", C.c_double),
                ("block_size", C.c_int64)]


assert DECISION_DT.itemsize == 104 and PREFILL_DT.itemsize == 32 and DECODE_DT.itemsize == 24

f = _L.kvx_schedule_batch
f.restype = C.c_int
f.argtypes = [C.POINTER(KvxPerfParams), C.POINTER(KvxSchedParams), _vp, _i64, _vp, _i64, _vp,
              _vp, _i64, _vp, _vp]


@dataclass
class PerfParams:
    """kvcsim::PerfModelParams defaults (proj/include/kvcsim/perf_model.hpp:13-26)."""
    alpha_mlp: float = 0.1
    beta_attn: float = 2.0e-6
    gamma_decode: float = 20.0
    delta_decode: float = 0.5
    epsilon_decode: float = 0.2
    kv_bytes_per_token: float = 327680.0
    link_bandwidth: float = 1.0e8
    load_bandwidth: float = 3.0e7
    prefill_chunk: int = 2048
    cpp_group_size: int = 1


def _dev_bytes(arr: np.ndarray, device) -> torch.Tensor:
    return torch.from_numpy(arr.view(np.uint8).reshape(-1).copy()).to(device)


def schedule_batch(perf: PerfParams, l_ttft_ms: float, l_tbt_ms: float, threshold: float,
                   block_size: int, now_ms: float, prefill: np.ndarray, decode: np.ndarray,
                   input_len: torch.Tensor, match_len: torch.Tensor, stream=None) -> np.ndarray:
    """prefill: PREFILL_DT records (instance order = match_len columns);
    decode: DECODE_DT records; input_len (n_req,) int64 and match_len
    (n_req, n_prefill) int64 on the GPU.  Returns DECISION_DT records."""
    dev = input_len.device
    p = KvxPerfParams(perf.alpha_mlp, perf.beta_attn, perf.gamma_decode, perf.delta_decode,
                      perf.epsilon_decode, perf.kv_bytes_per_token, perf.link_bandwidth,
                      perf.load_bandwidth, perf.prefill_chunk, perf.cpp_group_size)
    sp = KvxSchedParams(l_ttft_ms, l_tbt_ms, threshold, now_ms, block_size)
    # the snapshots, the result and its read-back all live on the launch stream
    # (the caching allocator then never recycles them while the kernel runs)
    ts = kvx._torch_stream(stream, dev)
    n_req = input_len.numel()
    with torch.cuda.stream(ts):
        d_pre = _dev_bytes(np.ascontiguousarray(prefill, dtype=PREFILL_DT), dev)
        d_dec = _dev_bytes(np.ascontiguousarray(decode, dtype=DECODE_DT), dev)
        out = torch.empty(max(n_req, 1) * DECISION_DT.itemsize, dtype=torch.uint8, device=dev)
        check(f(C.byref(p), C.byref(sp), d_pre.data_ptr(), len(prefill), d_dec.data_ptr(),
                len(decode), input_len.data_ptr(), match_len.data_ptr(), n_req, out.data_ptr(),
                kvx._stream(ts)))
        host = out.cpu().numpy()  # a copy on ts: ordered after the kernel, host waits
    return host[: n_req * DECISION_DT.itemsize].view(DECISION_DT)
