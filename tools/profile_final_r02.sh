set -x
export KEEP_REP=0
for n in 16 24 32 64; do bash tools/ncu_export.sh hh$n "bed_hh_kernel" 0 python tools/profile_cases.py $n; done
bash tools/ncu_export.sh bwd16 "bed_backward_kernel" 0 python tools/profile_cases.py 16
bash tools/ncu_export.sh pow16 "bed_power_kernel" 0 python tools/profile_cases.py 16 pow
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cases.csv \
    python tools/profile_cases.py > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv \
    python bench.py --steps 5 --warmup 3 --quick > gpurun_out/bench_under_ncu.json 2>&1
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
python bench.py --impl reference > gpurun_out/bench_final_ref.json 2> gpurun_out/bench_final_ref.err
tail -c 600 gpurun_out/bench_final.json
