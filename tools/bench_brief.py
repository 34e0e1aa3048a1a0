"""One-line digest of bench.py JSON lines (path time, steps/s, e2e, dominant kernel)."""
import json
import sys

for path in sys.argv[1:]:
    d = json.load(open(path))
    r = d.get("roofline", {})
    print(d["config"]["workload"], f"{d['ms_per_step']:.3f} ms", f"{d['value']:.1f} {d['unit']}",
          "e2e", f"{d['e2e']['ms_per_step']:.2f} ms" if d.get("e2e", {}).get("ms_per_step") else d.get("e2e"),
          "| kernel", (r.get("kernel") or "")[:24], f"{1000 * (r.get('avg_launch_ms') or 0):.1f} us",
          f"frac {r.get('frac') or 0:.3f}", "| clocks", d.get("clocks", {}).get("sm_mhz"), d.get("clocks", {}).get("reasons"))
