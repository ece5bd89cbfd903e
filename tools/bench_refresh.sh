# final bench line + reference arm + launch lists (outputs in gpurun_out/)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cases.csv \
    python tools/profile_cases.py > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv \
    python bench.py --steps 5 --warmup 3 --quick > gpurun_out/bench_under_ncu.json 2>&1
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
python bench.py --impl reference > gpurun_out/bench_final_ref.json 2> gpurun_out/bench_final_ref.err
tail -c 300 gpurun_out/bench_final.json
