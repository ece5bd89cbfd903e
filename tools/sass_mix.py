"""Dynamic instruction mix of an ncu SASS export: warp-level executed
instructions per opcode, per matrix (python tools/sass_mix.py <sass.csv.gz>
<matrices>)."""
import csv
import gzip
import sys
from collections import Counter

rows = list(csv.reader(gzip.open(sys.argv[1], "rt")))
hdr, data = rows[1], rows[2:]
isrc, iexe = hdr.index("Source"), hdr.index("Instructions Executed")
mats = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
cnt = Counter()
for r in data:
    try:
        n = int(r[iexe])
    except ValueError:
        continue
    op = r[isrc].strip().split()
    if not op:
        continue
    k = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
    cnt[k.split(".")[0]] += n
tot = sum(cnt.values())
print(f"total warp-instructions {tot}, per matrix {tot / mats:.1f} (x32 threads)")
for k, v in cnt.most_common(30):
    print(f"  {k:12s} {v / mats:9.2f}  {100 * v / tot:5.1f}%")
