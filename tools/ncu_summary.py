"""Condense ncu exports (gpurun_out/<name>.raw.csv / .details.csv) into
profiles/<round>_ncu_summary.md and profiles/ncu_summary.json (the traffic
figure bench.py reports)."""
import csv
import json
import os
import sys

OUT = "profiles"
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "smsp__thread_inst_executed_per_inst_executed.ratio",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__warps_eligible.avg.per_cycle_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__pcsamp_warps_issue_stalled_no_instructions",
    "smsp__pcsamp_warps_issue_stalled_barrier",
    "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle",
    "smsp__pcsamp_sample_count",
]


def raw(name):
    path = os.path.join("gpurun_out", f"{name}.raw.csv")
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    vals = rows[2]
    d = {}
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            d[k] = (vals[i], units[i])
    d["kernel"] = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else name
    return d


def main(round_tag, names, headline=None):
    md = [f"# ncu summaries, {round_tag}", "",
          "One `ncu --set full --clock-control none` capture per kernel (cold cache, serialised; "
          "compare shares, not absolutes).  Source: gpurun_out/<name>.raw.csv.", ""]
    js = {}
    jpath = os.path.join(OUT, "ncu_summary.json")
    if os.path.exists(jpath):
        js = json.load(open(jpath))
    for name in names:
        d = raw(name)
        md.append(f"## {name}: `{d['kernel'][:110]}`")
        md.append("")
        md.append("| metric | value | unit |")
        md.append("|---|---|---|")
        for k in KEYS:
            if k in d:
                md.append(f"| {k} | {d[k][0]} | {d[k][1]} |")
        md.append("")
        rb = float(d["dram__bytes_read.sum"][0].replace(",", "")) if "dram__bytes_read.sum" in d else 0
        wb = float(d["dram__bytes_write.sum"][0].replace(",", "")) if "dram__bytes_write.sum" in d else 0
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rb *= scale.get(d.get("dram__bytes_read.sum", ("", "byte"))[1], 1)
        wb *= scale.get(d.get("dram__bytes_write.sum", ("", "byte"))[1], 1)
        key = d["kernel"].split("(")[0].replace("void ", "").replace("bed::", "").replace(" ", "")
        js[key] = {"profile": name, "round": round_tag, "dram_bytes_per_launch": rb + wb,
                   "duration": d.get("gpu__time_duration.sum")}
    open(os.path.join(OUT, f"{round_tag}_ncu_summary.md"), "w").write("\n".join(md) + "\n")
    json.dump(js, open(jpath, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
