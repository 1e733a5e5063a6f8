"""Drop-in proof on the GPU: the reference's own engine / conductor / acceptance
code, compiled against include/kvcsim/kvcache.hpp and linked with the
GPU-backed libkvcsim_gpu.so instead of the reference's kvcache.cpp
(oracle/dropin.mk), must reproduce the pure-reference build exactly:

* tests/dropin/replay_main.cpp -- six cluster scenarios (LRU/LFU/LengthAware,
  bounded and unbounded pools, migrations incl. aborts): every
  SimReport::to_json_string byte-identical to tests/golden/replay_reports.txt;
* the reference's acceptance suite (proj/tests/acceptance_main.cpp): the same
  PASS/SKIP lines as tests/golden/acceptance_ref.txt.

The binaries are built in the build container (they need /root/reference) and
travel to the GPU box with the snapshot; the tests skip if they are absent.
"""
import os
import re
import subprocess

import pytest

from conftest import GOLDEN, ROOT

REF_DIR = os.path.join(ROOT, "oracle", "_ref")


def _bin(name):
    p = os.path.join(REF_DIR, name)
    if not os.path.exists(p):
        pytest.skip(f"{p} not built (make -f oracle/dropin.mk in the build container)")
    return p


def _norm(txt):
    return [re.sub(r"[0-9]+\.[0-9]+s", "", ln) for ln in txt.splitlines()]


def test_ref_replay_matches_golden_cpu():
    """CPU: the pure-reference build reproduces the committed golden (stability)."""
    out = subprocess.run([_bin("ref_replay")], capture_output=True, text=True, check=True,
                         timeout=300).stdout
    assert out == open(os.path.join(GOLDEN, "replay_reports.txt")).read()


@pytest.mark.gpu
def test_dropin_replay_byte_identical(kvx):
    out = subprocess.run([_bin("dropin_replay")], capture_output=True, text=True, check=True,
                         timeout=900).stdout
    want = open(os.path.join(GOLDEN, "replay_reports.txt")).read()
    got_l, want_l = out.splitlines(), want.splitlines()
    assert len(got_l) == len(want_l)
    for g, w in zip(got_l, want_l):
        assert g == w, g.split(" ", 1)[0]


@pytest.mark.gpu
def test_dropin_acceptance_suite(kvx):
    r = subprocess.run([_bin("dropin_acceptance")], capture_output=True, text=True, timeout=1800)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    got = _norm(r.stdout)
    want = _norm(open(os.path.join(GOLDEN, "acceptance_ref.txt")).read())
    assert got == want
