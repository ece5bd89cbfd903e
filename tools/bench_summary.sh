#!/bin/bash
# print a compact view of a bench.py JSON line
python - "$1" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("HEAD %.3f G/s  %.3f ms  frac %.3f  steps %.2f  clocks %s" % (d["value"]/1e9, d["ms_per_step"], d["roofline"]["frac"], d["config"]["mean_double_steps"], d.get("clocks")))
if "e2e" in d: print("E2E %.1f M/s" % (d["e2e"]["value"]/1e6))
if "cpu_baseline" in d: print("CPU %.1f M/s (%s cores)" % (d["cpu_baseline"]["value"]/1e6, d["cpu_baseline"]["cores"]))
for r in d.get("other_configs", []):
    print("  n=%-2d b=%-8d %-6s %8.3f ms %10.2f M/s frac %.4f steps %.1f" % (r["n"], r["batch"], r["mode"], r["ms"], r["value"]/1e6, r["roofline_frac"], r["mean_double_steps"]))
PY
