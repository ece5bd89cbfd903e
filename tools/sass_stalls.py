"""Hot instructions of an ncu SASS source export (tools/ncu_export.sh writes
gpurun_out/<name>.sass.csv.gz): python tools/sass_stalls.py <file> [top] [lo-hi]

Prints the instructions with the most warp-stall samples, with the stall
reason columns that dominate them, plus samples summed per 256-byte region."""
import csv
import gzip
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
rows = list(csv.reader(gzip.open(path, "rt")))
hdr = rows[1]
data = rows[2:]
ia, isrc, isamp = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
iexe = hdr.index("Instructions Executed")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") or "Stall" in h and i > isamp + 1]
base = int(data[0][ia], 16)
recs = []
for r in data:
    try:
        s = float(r[isamp])
    except ValueError:
        continue
    recs.append((s, int(r[ia], 16) - base, r[isrc].strip(), r[iexe]))
tot = sum(r[0] for r in recs)
print(f"total samples {tot:.0f}, instructions {len(recs)}")
for s, off, src, ex in sorted(recs, reverse=True)[:top]:
    print(f"{s:7.0f} {100*s/tot:5.1f}%  +0x{off:05x}  exec {ex:>9s}  {src}")
# region histogram
reg = {}
for s, off, src, ex in recs:
    reg[off // 1024] = reg.get(off // 1024, 0) + s
print("samples per 1 KB of code:")
for k in sorted(reg):
    if reg[k] > 0.01 * tot:
        print(f"  +0x{k*1024:05x}: {100*reg[k]/tot:5.1f}%")

# stall reasons summed over an address range: [lo-hi] as hex offsets
if len(sys.argv) > 3:
    lo, hi = (int(x, 16) for x in sys.argv[3].split("-"))
    cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    sums = {hdr[i]: 0.0 for i in cols}
    n_ex = 0
    for r in data:
        off = int(r[ia], 16) - base
        if lo <= off < hi:
            for i in cols:
                try:
                    sums[hdr[i]] += float(r[i])
                except ValueError:
                    pass
            try:
                n_ex += int(r[iexe])
            except ValueError:
                pass
    print(f"range +0x{lo:x}-+0x{hi:x}: warp-instructions executed {n_ex}")
    for k, v in sorted(sums.items(), key=lambda kv: -kv[1])[:10]:
        print(f"  {k:28s} {v:8.0f}")
