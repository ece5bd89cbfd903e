L=paper_2207_04228_b200/_lib/libbed200.so
# A/B two builds of libbed200.so (copied to _ab/old.so, _ab/new.so) under an ncu launch list
for v in old new old new; do cp _ab/$v.so $L; echo "== $v"; ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"bed_hh|bed_power_kernel|bed_small" python tools/profile_cases.py 16 24 32 pow 2>&1 | grep -E "bed_|duration" | paste - - | awk '{print $1, $NF}' | sed 's/(.*//' ; done
