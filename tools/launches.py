"""Summarise an ncu --csv launch list (gpu__time_duration.sum): bed_ kernels only.
usage: python tools/launches.py gpurun_out/launches.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = {k: j for j, k in enumerate(rows[start])}
for r in rows[start + 1:]:
    k = r[h["Kernel Name"]]
    if "bed_" in k:
        name = k.split("(")[0].replace("void bed::", "")
        print(f"{name:40s} grid {r[h['Grid Size']]:>14s} blk {r[h['Block Size']]:>12s} {float(r[h['Metric Value']])/1e3:9.1f} us")
