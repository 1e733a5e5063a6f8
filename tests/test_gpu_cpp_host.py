"""A C++ host program drives the hot path through the C ABI alone
(examples/kvx_demo.cpp): hash -> prefix match -> layer-wise stream -> verify."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_cpp_host_demo(kvx):
    exe = os.path.join(ROOT, "examples", "kvx_demo")
    if not os.path.exists(exe):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "examples")], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "kvx_demo OK" in r.stdout
