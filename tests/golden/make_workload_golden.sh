#!/bin/bash
# Pins the synthetic Config 1/2/5 block selections to the reference's own
# generate_workload (proj/src/trace.cpp:163-222): builds workload_gen.cpp
# against the UNMODIFIED reference trace.cpp in /tmp and writes
# tests/golden/workload_ids.npz.  Build container only (needs /root/reference).
set -e
HERE="$(cd "$(dirname "$0")" && pwd)"
REF=${REF:-/root/reference/proj}
JSON_DIR=$(dirname "$(ls /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann/json.hpp)")
OUT=/tmp/kvx_workload_gen
g++ -O2 -std=c++20 -w -include array -I"$REF/include" -I"$JSON_DIR/.." -I"$JSON_DIR" \
    -o "$OUT" "$HERE/workload_gen.cpp" "$REF/src/trace.cpp"
python - "$OUT" "$HERE/workload_ids.npz" <<'PY'
import subprocess, sys
import numpy as np
gen, out = sys.argv[1], sys.argv[2]
arrays = {}
for name, args in {"c2_bs16": ["64", "8192", "0.5", "16"], "c1_bs16": ["1", "8192", "0.5", "16"],
                   "c2_bs64": ["64", "8192", "0.5", "64"], "c2_bs512": ["8", "8192", "0.5", "512"],
                   "c2_r03": ["5", "8000", "0.3", "16"]}.items():
    lines = subprocess.run([gen, *args], capture_output=True, text=True, check=True).stdout.split("\n")
    rows = [np.array(ln.split()[1:], dtype=np.int64) for ln in lines if ln.strip()]
    arrays[name] = np.stack(rows)
    arrays[name + "_args"] = np.array([float(a) for a in args])
np.savez_compressed(out, **arrays)
print("wrote", out, {k: v.shape for k, v in arrays.items() if not k.endswith("_args")})
PY
