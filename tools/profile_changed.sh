set -x
export KEEP_REP=0
bash tools/ncu_export.sh small8 "bed_small_kernel" 0 python tools/profile_cases.py 8
for n in 32 64; do
  bash tools/ncu_export.sh hh$n "bed_hh_kernel" 0 python tools/profile_cases.py $n
  bash tools/ncu_export.sh qr$n "bed_qr_kernel" 0 python tools/profile_cases.py $n
  bash tools/ncu_export.sh ft$n "bed_fold_tma_kernel" 0 python tools/profile_cases.py $n
done
bash tools/ncu_export.sh bwdtc64 "bed_backward_tc_kernel" 0 python tools/profile_cases.py 64
bash tools/ncu_export.sh scatsmall4 "bed_scatter_small_kernel" 0 python tools/profile_cases.py 4 scatpow
