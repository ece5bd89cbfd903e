"""Print the headline metrics and the top warp-stall reasons of an ncu raw
export: python tools/ncu_quick.py gpurun_out/<name>.raw.csv [more...]"""
import csv
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.sum", "launch__registers_per_thread", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_blocks",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__warps_eligible.avg.per_cycle_active",
]

for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    print(f"== {path}: {vals[hdr.index('Kernel Name')][:70]}")
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            print(f"  {k:70s} {vals[i]:>14s} {units[i]}")
    stalls = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warp_latency_issue_stalled_") or (
                h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")):
            try:
                stalls.append((float(vals[i].replace(",", "")), h))
            except ValueError:
                pass
    stalls.sort(reverse=True)
    for v, h in stalls[:10]:
        print(f"  stall {h:80s} {v:12.1f}")
