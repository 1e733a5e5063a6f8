"""Summarise ncu outputs brought back in gpurun_out/ into profiles/.

    python profiles/summarize_ncu.py r01

Reads gpurun_out/launches_<tag>.csv (gpu__time_duration per launch) and the
--set full reports gpurun_out/prof_*_<tag>.ncu-rep, writes
profiles/ncu_<tag>.md (human summary) and merges per-launch DRAM traffic into
profiles/ncu_traffic.json (read by bench.py for roofline.traffic).
"""
import collections
import csv
import io
import json
import re
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes.sum.per_second",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "lts__t_sector_hit_rate.pct", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6,
         "usecond": 1e-6, "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9}


def launches(tag):
    path = os.path.join(OUT, f"launches_{tag}.csv")
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0) * 1e6  # -> us
        agg[r[ki].split("(")[0].replace("kvx::<unnamed>::", "")].append(v)
    return agg


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        name = vals[h.index("Kernel Name")].split("(")[0].replace("kvx::<unnamed>::", "") \
            .replace("unnamed>::", "")
        d = {"kernel": re.sub(r"^void |<.*>$", "", name)}  # copy_lsu_kernel<unsigned int> -> copy_lsu_kernel
        for m in METRICS:
            if m in h:
                i = h.index(m)
                d[m] = f"{vals[i]} {units[i]}".strip()
                try:
                    d[m + ":value"] = float(vals[i].replace(",", "")) * SCALE.get(units[i], 1.0)
                except ValueError:
                    pass
        out.append(d)
    return out


def main(tag):
    lines = [f"# ncu summary, round tag {tag}", ""]
    agg = launches(tag)
    tot = sum(sum(v) for v in agg.values())
    lines += ["## Launch list (bench.py small transfer config; `gpu__time_duration.sum`, "
              "serialised, cold-cache -- compare shares)", "",
              "| kernel | launches | avg us | total ms | share |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        lines.append(f"| {k} | {len(v)} | {sum(v)/len(v):.1f} | {sum(v)/1e3:.2f} | "
                     f"{sum(v)/tot:.3f} |")
    traffic_path = os.path.join(PROF, "ncu_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    for rep in sorted(f for f in os.listdir(OUT) if f.endswith(f"_{tag}.ncu-rep")):
        lines += ["", f"## `--set full`: {rep}", ""]
        for d in raw(os.path.join(OUT, rep)):
            lines.append(f"### {d['kernel']}")
            for m in METRICS:
                if m in d:
                    lines.append(f"- `{m}` = {d[m]}")
            rd = d.get("dram__bytes_read.sum:value")
            wr = d.get("dram__bytes_write.sum:value")
            if rd is not None and wr is not None:
                lines.append(f"- DRAM traffic per launch = {rd + wr:.4g} B")
                traffic[d["kernel"]] = rd + wr
            lines.append("")
    with open(os.path.join(PROF, f"ncu_{tag}.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(traffic_path, "w") as f:
        json.dump(traffic, f, indent=1, sort_keys=True)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
