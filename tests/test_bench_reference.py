"""CPU: the reference arm of bench.py (the oracle port of the byte path timed
on host threads) prints the contract's JSON line -- `impl`, the same metric /
unit as the kvx arm, a `cpu_baseline` describing the run and a zero-copy
`e2e` -- and exits 0 without a GPU."""
import json
import os
import subprocess
import sys

from conftest import ROOT


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "2", "--warmup", "1"],
                         capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["impl"] == "reference"
    assert line["unit"] == "GB/s" and line["higher_is_better"] is True
    assert line["metric"].startswith("KVCache layer-wise transfer GB/s")
    assert line["steps"] == 2 and line["warmup"] == 1 and line["value"] > 0
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": "GB/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    # the same config object as the kvx arm at N=1 (the driver pairs the two lines)
    cfg = line["config"]
    assert cfg["workload"].startswith("config2") and cfg["mode"] == "local_fused"
    assert cfg["requests"] == 64 and cfg["layers_per_chunk"] == 1
    assert "Config 2 sample" in cb["sample"] and cb["cpu_model"]
