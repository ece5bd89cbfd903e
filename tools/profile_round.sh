#!/bin/bash
# One ncu --set full capture per final kernel (tools/ncu_export.sh) and the
# launch list of the cases and of a short bench run.  Outputs in gpurun_out/;
# summarise with: python tools/ncu_summary.py <round> <names...>
set -x
export KEEP_REP=${KEEP_REP:-0}
bash tools/ncu_export.sh small4 "bed_small_kernel" 0 python tools/profile_cases.py 4
bash tools/ncu_export.sh small8 "bed_small_kernel" 0 python tools/profile_cases.py 8
for n in 16 24 32 64; do
  bash tools/ncu_export.sh hh$n "bed_hh_kernel" 0 python tools/profile_cases.py $n
  bash tools/ncu_export.sh qr$n "bed_qr_kernel" 0 python tools/profile_cases.py $n
  bash tools/ncu_export.sh ft$n "bed_fold_tma_kernel" 0 python tools/profile_cases.py $n
done
bash tools/ncu_export.sh bwd16 "bed_backward_kernel" 0 python tools/profile_cases.py 16
bash tools/ncu_export.sh bwd64 "bed_backward_tc_kernel" 0 python tools/profile_cases.py 64
bash tools/ncu_export.sh pow16 "bed_power_kernel" 0 python tools/profile_cases.py 16 pow
bash tools/ncu_export.sh scat16 "bed_scatter_kernel" 0 python tools/profile_cases.py scat
bash tools/ncu_export.sh powf4 "bed_small_kernel" 0 python tools/profile_cases.py 4 powf
bash tools/ncu_export.sh powf16 "bed_fold_tma_kernel" 0 python tools/profile_cases.py 16 powf
bash tools/ncu_export.sh scatpow4 "bed_small_kernel" 0 python tools/profile_cases.py 4 scatpow
bash tools/ncu_export.sh scatsmall4 "bed_scatter_small_kernel" 0 python tools/profile_cases.py 4 scatpow
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cases.csv \
    python tools/profile_cases.py > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv \
    python bench.py --steps 5 --warmup 3 --quick > gpurun_out/bench_under_ncu.json 2>&1
