"""One-screen summary of a bench.py JSON line: python tools/bench_brief.py FILE"""
import json
import sys

for line in open(sys.argv[1]):
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    print("value %.4g %s  ms/step %.5f  frac %.3f  step_ms %s" % (
        d["value"], d["unit"], d["ms_per_step"], d.get("roofline", {}).get("frac", 0), d.get("step_ms")))
    for k in ("time_loop", "o1280_strong", "e2e", "e2e_time_loop"):
        r = d.get(k)
        if r:
            print(f"  {k}: value {r.get('value', 0):.4g} ms/step {r.get('ms_per_step')} frac {r.get('roofline_frac')}")
    print("  clocks", d.get("clocks"))
