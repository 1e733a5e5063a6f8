"""Tabulate the Config 5 sweep (gpurun_out/c5/*.json) as markdown.
python profiles/c5_table.py [dir] > profiles/r01/c5_sweep.md"""
import glob
import json
import os
import re
import sys

d = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/c5"
rows = []
for f in sorted(glob.glob(os.path.join(d, "*.json"))):
    m = re.match(r"n(\d)_bs(\d+)_dt(\d)", os.path.basename(f))
    lines = [ln for ln in open(f).read().splitlines() if ln.startswith("{")]
    if not m or not lines:
        continue
    j = json.loads(lines[-1])
    r = j.get("roofline") or {}
    link = j.get("link") or {}
    rows.append((int(m.group(1)), int(m.group(2)), int(m.group(3)), j["value"],
                 r.get("achieved"), r.get("frac"), link.get("frac"), j["parity"]["mismatched_words"],
                 j["config"].get("mode")))
rows.sort()
print("| N | block size | KV dtype | slab | payload GB/s | dominant kernel GB/s | frac (HBM) | "
      "frac (link) | mismatches | mode |")
print("|---|---|---|---|---|---|---|---|---|---|")
for n, bs, dt, v, ach, fr, lf, bad, mode in rows:
    dtn = "fp8" if dt == 1 else "fp16/bf16"
    slab = bs * 8 * 128 * dt
    print(f"| {n} | {bs} | {dtn} | {slab // 1024} KiB | {v:.1f} | {ach:.1f} | {fr:.3f} | "
          f"{'' if lf is None else f'{lf:.3f}'} | {bad} | {mode} |")
