"""Opcode histogram of the largest loop (backward branch span) of a kernel's
SASS: python tools/sass_loop.py <obj-or-cubin> <mangled-name-regex>."""
import re
import subprocess
import sys
from collections import Counter

obj, pat = sys.argv[1], sys.argv[2]
names = re.findall(r"Function : (\S+)", subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout)
fn = next(n for n in names if re.search(pat, n))
out = subprocess.run(["cuobjdump", "-sass", "-fun", fn, obj], capture_output=True, text=True).stdout
ins = []
for line in out.splitlines():
    m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
loops = []
for addr, txt in ins:
    m = re.search(r"BRA(?:\.\S+)?\s+(?:!?U?P\d+,\s*)?0x([0-9a-f]+)", txt)
    if m:
        tgt = int(m.group(1), 16)
        if tgt < addr:
            loops.append((tgt, addr))
loops.sort(key=lambda x: x[0] - x[1])
nshow = int(sys.argv[3]) if len(sys.argv) > 3 else 1
print(f"{fn[:60]}: total {len(ins)}")
for lo, hi in loops[:nshow]:
    body = [t for a, t in ins if lo <= a <= hi]
    ops = Counter()
    for t in body:
        tok = t.split()
        o = tok[1] if tok[0].startswith("@") else tok[0]
        ops[o.split(".")[0]] += 1
    print(f"  loop [{lo:#x},{hi:#x}] {len(body)} instr")
    print("    " + " ".join(f"{o}:{c}" for o, c in ops.most_common(30)))
