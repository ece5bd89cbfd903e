"""Summarise an ncu --page source --print-source sass CSV: hottest
instruction windows by executed instructions and by stall samples, plus the
opcode mix."""
import csv
import gzip
import sys
from collections import Counter

path = sys.argv[1]
topk = int(sys.argv[2]) if len(sys.argv) > 2 else 40
W = int(sys.argv[3]) if len(sys.argv) > 3 else 32
op = gzip.open if path.endswith(".gz") else open
with op(path, "rt") as f:
    rows = list(csv.reader(f))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
tot_exec = sum(int(r[idx["Instructions Executed"]] or 0) for r in data)
tot_samp = sum(int(r[idx["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
print(f"{len(data)} sass lines, executed warp-instr {tot_exec:,}, stall samples {tot_samp:,}")
for key in ("Instructions Executed", "Warp Stall Sampling (All Samples)"):
    wins = []
    for s in range(0, len(data), W):
        v = sum(int(r[idx[key]] or 0) for r in data[s:s + W])
        wins.append((v, s))
    wins.sort(reverse=True)
    tot = tot_exec if key.startswith("Instr") else tot_samp
    print(f"\n== top windows by {key}")
    for v, s in wins[:10]:
        ops = " ".join(r[idx["Source"]].split()[0] for r in data[s:s + W] if r[idx["Source"]].strip())
        print(f"{100.0*v/max(tot,1):5.1f}% @{s:5d}: {ops[:200]}")
mix = Counter()
for r in data:
    t = r[idx["Source"]].split()
    if not t:
        continue
    o = t[1] if t[0].startswith("@") else t[0]
    mix[o.split(".")[0]] += int(r[idx["Instructions Executed"]] or 0)
print("\n== opcode mix (executed warp-instr)")
print("  ".join(f"{o}:{100.0*v/tot_exec:.1f}%" for o, v in mix.most_common(topk)))
