S=/usr/local/cuda/bin/compute-sanitizer
echo "== memcheck"; timeout 900 $S --tool memcheck python tools/sanitize_cases.py 2>&1 | tail -2
echo "== racecheck"; timeout 1200 $S --tool racecheck --racecheck-report hazard python tools/sanitize_cases.py > gpurun_out/race.log 2>&1; tail -2 gpurun_out/race.log
grep -o "in [a-z_]*\.cuh:[0-9]*" gpurun_out/race.log | sort | uniq -c | sort -rn | head -20
grep -B2 "Race reported" gpurun_out/race.log | grep -o "void [a-z_:]*bed_[a-z_]*_kernel" | sort | uniq -c
echo "== synccheck"; timeout 900 $S --tool synccheck python tools/sanitize_cases.py 2>&1 | tail -2
