#!/bin/bash
# usage: tools/ncu_export.sh <name> <kernel-regex> <launch-skip> <cmd...>
# Captures one launch with --set full, exports raw + source CSV next to it,
# and removes the (large) .ncu-rep unless KEEP_REP=1.
name=$1; kre=$2; skip=$3; shift 3
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k "regex:$kre" -s "$skip" -c 1 \
    -o "gpurun_out/$name" -f "$@" > "gpurun_out/$name.ncu.log" 2>&1
ncu -i "gpurun_out/$name.ncu-rep" --page raw --csv > "gpurun_out/$name.raw.csv" 2>/dev/null
ncu -i "gpurun_out/$name.ncu-rep" --page details --csv > "gpurun_out/$name.details.csv" 2>/dev/null
ncu -i "gpurun_out/$name.ncu-rep" --page source --csv --print-source sass > "gpurun_out/$name.sass.csv" 2>/dev/null
gzip -f "gpurun_out/$name.sass.csv"
[ "$KEEP_REP" = "1" ] || rm -f "gpurun_out/$name.ncu-rep"
ls -la gpurun_out/ | grep "$name"
