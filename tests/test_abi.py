"""CPU tests of the C-ABI boundary: libkvx.so loads, exports every entry point
include/kvx.h declares, its scalar chain_hash matches the reference's golden
vectors, and compute entry points fail loudly (no CPU fallback) without a GPU."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest
import torch

from conftest import ROOT, golden

LIB = os.path.join(ROOT, "paper_2407_00079_b200", "libkvx.so")
HDR = os.path.join(ROOT, "include", "kvx.h")
# every C header under include/ and the library that must export it
C_HEADERS = {"kvx.h": LIB,
             "kvcsim_c.h": os.path.join(ROOT, "paper_2407_00079_b200", "libkvcsim_gpu.so")}


def _ensure_built():
    if not all(os.path.exists(p) for p in C_HEADERS.values()):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2407_00079_b200", "csrc")],
                       check=True)


def declared_symbols(header=HDR):
    txt = open(header).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b((?:kvx|kvcsim)_[a-z0-9_]+)\s*\(", txt)))


def test_every_c_header_is_covered():
    hdrs = sorted(f for f in os.listdir(os.path.join(ROOT, "include")) if f.endswith(".h"))
    assert hdrs == sorted(C_HEADERS)


@pytest.mark.parametrize("header", sorted(C_HEADERS))
def test_each_header_exported(header):
    _ensure_built()
    lib = C_HEADERS[header]
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT ((?:kvx|kvcsim)_[a-z0-9_]+)\b", out))
    syms = declared_symbols(os.path.join(ROOT, "include", header))
    assert syms and not [s for s in syms if s not in exported]
    handle = C.CDLL(lib)
    for s in syms:
        getattr(handle, s)


def test_header_declares_the_survey_minimum():
    syms = set(declared_symbols())
    # SURVEY.md 8(b) "C-ABI must export (minimum)"
    for s in ["kvx_chain_hash_batch", "kvx_index_create", "kvx_index_destroy",
              "kvx_index_insert", "kvx_index_erase", "kvx_match_prefix_batch",
              "kvx_pool_create", "kvx_gather", "kvx_transfer_submit", "kvx_transfer_wait",
              "kvx_scatter", "kvx_last_error"]:
        assert s in syms, s


def test_library_exports_every_declared_symbol():
    _ensure_built()
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (kvx_[a-z0-9_]+)\b", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    lib = C.CDLL(LIB)
    for s in declared_symbols():
        getattr(lib, s)


def test_library_is_sm100a():
    _ensure_built()
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_scalar_chain_hash_golden():
    _ensure_built()
    lib = C.CDLL(LIB)
    lib.kvx_chain_hash.restype = C.c_int64
    lib.kvx_chain_hash.argtypes = [C.c_int64, C.c_uint64]
    g = golden("chain_hash.npz")
    got = np.array([lib.kvx_chain_hash(int(p), int(c)) for p, c in zip(g["prev"], g["content"])],
                   dtype=np.int64)
    assert np.array_equal(got, g["out"])


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks behaviour without a GPU")
def test_no_cpu_fallback_without_gpu():
    _ensure_built()
    import paper_2407_00079_b200 as pkg
    with pytest.raises(pkg.KvxError):
        pkg.BlockIndex(0, 16)
    with pytest.raises(pkg.KvxError):
        pkg.KVPool(2, 16, 8, 128, 2, 4, 0)


def test_validation_errors_map_to_einval():
    _ensure_built()
    import paper_2407_00079_b200 as pkg
    # empty prefill pool -> ValidationError (conductor.cpp:59-61), checked before any device work
    with pytest.raises(pkg.ValidationError):
        pkg.kvx.check(pkg.kvx._L.kvx_match_prefix_batch(None, None, 0, None, None, 1, None, None,
                                                        None, None))
    with pytest.raises(pkg.ValidationError):
        pkg.kvx.check(pkg.kvx._L.kvx_set_copy_impl(7))
