set -x
python tools/quick_time.py > gpurun_out/quick.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_cases.py > /dev/null 2>&1
bash tools/ncu_export.sh small4 bed_small_kernel 0 python tools/profile_cases.py 4
