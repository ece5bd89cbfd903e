#!/bin/bash
# per-kernel device times of tools/profile_cases.py (ncu launch list)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python tools/profile_cases.py "$@" > /dev/null 2>&1
python tools/launches.py gpurun_out/launches.csv
