# PDL timing cross-check: C2-shaped local fused step, events vs host wall clock with device sync,
# and a full verify of every destination word after the timed steps.
import subprocess, json, sys, os
for pdl in ("1", "0"):
    env = dict(os.environ, KVX_STREAM_PDL=pdl)
    out = subprocess.run([sys.executable, "bench.py", "--no-match", "--no-cpu-baseline", "--no-e2e"],
                         capture_output=True, text=True, env=env).stdout
    d = json.loads([l for l in out.splitlines() if l.startswith("{")][-1])
    print(f"PDL={pdl}: value={d['value']:.1f} GB/s event ms/step={d['ms_per_step']:.3f} "
          f"host wall ms/step={d['host_wall_ms_per_step']:.3f} roof={d['roofline']['achieved']:.0f}")
