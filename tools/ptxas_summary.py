"""Summarise ptxas -v logs: registers, stack frame and spills per kernel."""
import glob
import re
import subprocess
import sys

for path in sorted(glob.glob(sys.argv[1] if len(sys.argv) > 1 else "paper_2207_04228_b200/_build/*.ptxas.log")):
    cur = None
    rows = []
    for line in open(path):
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            cur = m.group(1)
            try:
                cur = subprocess.run(["c++filt", cur], capture_output=True, text=True).stdout.strip()
                cur = re.sub(r"\(.*", "", cur).replace("bed::", "")
            except Exception:
                pass
            rec = {"name": cur}
            rows.append(rec)
        m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m and rows:
            rows[-1]["stack"], rows[-1]["spill_st"], rows[-1]["spill_ld"] = map(int, m.groups())
        m = re.search(r"Used (\d+) registers", line)
        if m and rows:
            rows[-1]["regs"] = int(m.group(1))
    for r in rows:
        print(f"{r['name']:<60} regs={r.get('regs')} stack={r.get('stack')} spill={r.get('spill_st')}/{r.get('spill_ld')}")
