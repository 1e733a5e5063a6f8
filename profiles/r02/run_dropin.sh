#!/bin/bash
# r02: drop-in latency -- the reference engine relinked on libkvcsim_gpu.so vs the pure reference
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
python - <<'PY'
import os, subprocess, time
env = {**os.environ, "KVCSIM_GPU_STATS": "1"}
res = {}
for b in ["ref_replay", "dropin_replay", "ref_acceptance", "dropin_acceptance"]:
    best = None
    for rep in range(3):
        t0 = time.perf_counter()
        r = subprocess.run([f"oracle/_ref/{b}"], capture_output=True, text=True, env=env)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    open(f"gpurun_out/{b}.out", "w").write(r.stdout)
    res[b] = best
    print(f"{b}: rc={r.returncode} best wall {best:.3f} s  {r.stderr.strip().splitlines()[-1] if r.stderr.strip() else ''}")
print("replay reports identical:", open("gpurun_out/ref_replay.out").read() == open("gpurun_out/dropin_replay.out").read())
PY
