"""Print the key numbers of bench JSON lines: python profiles/show.py f1.json ..."""
import json
import sys

for f in sys.argv[1:]:
    lines = [ln for ln in open(f).read().splitlines() if ln.startswith("{")]
    if not lines:
        print(f, "no JSON line")
        continue
    d = json.loads(lines[-1])
    r = d.get("roofline") or {}
    print(f"{f}: value={d['value']:.1f} {d['unit']} ms/step={d['ms_per_step']:.2f} "
          f"n={d['n_gpus']} mode={d['config'].get('mode')} e2e={(d.get('e2e') or {}).get('value')}")
    print(f"   roof {r.get('kernel')} bound={r.get('bound')} achieved={r.get('achieved', 0):.1f} "
          f"peak={r.get('peak')} frac={r.get('frac', 0):.3f} launch_ms={r.get('avg_launch_ms', 0):.4f}")
    if d.get("link"):
        print(f"   link {json.dumps(d['link'])}")
    print(f"   parity={d['parity']['mismatched_words']} clocks={d['clocks']} launches={d['gpu_launches']}")
    if d.get("cpu_baseline"):
        print(f"   cpu {d['cpu_baseline']['value']:.2f} {d['cpu_baseline']['unit']} cores={d['cpu_baseline']['cores']}")
    m = d.get("match")
    if m:
        print(f"   match {m['value']:.3e} blocks/s ms={m['ms_per_step']:.4f} "
              + " ".join(f"{k}={v['avg_ms']:.4f}ms" for k, v in m['kernels'].items()))
