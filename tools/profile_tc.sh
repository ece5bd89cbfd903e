#!/bin/bash
# ncu --set full captures of the tcgen05 kernels (n = 64) and a launch list of
# the cases with them; summarise with tools/ncu_summary.py.
set -x
export KEEP_REP=${KEEP_REP:-0}
bash tools/ncu_export.sh bwdtc64 "bed_backward_tc_kernel" 0 python tools/profile_cases.py 64
bash tools/ncu_export.sh powtc64 "bed_power_tc_kernel" 0 python tools/profile_cases.py 64 pow
bash tools/ncu_export.sh scattc64 "bed_scatter_tc_kernel" 0 python tools/profile_cases.py scat
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_tc.csv \
    python tools/profile_cases.py 64 > /dev/null 2>&1
BED_TC=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_notc.csv \
    python tools/profile_cases.py 64 > /dev/null 2>&1
