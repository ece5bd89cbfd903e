# A/B two builds of libbed200.so (copied to _ab/old.so, _ab/new.so) under an ncu launch list:
#   bash tools/ab_kernels.sh [kernel-regex] [profile_cases args...]
L=paper_2207_04228_b200/_lib/libbed200.so
K=${1:-bed_}; shift
for v in old new old new; do cp _ab/$v.so $L; echo "== $v"
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$K" python tools/profile_cases.py "$@" 2>&1 \
    | grep -E "^  [a-z_]+.*\(|duration" | sed -E 's/^  (void )?([a-z_0-9]+<[^>]*>).*/\2/' | paste - - | awk '{print $1, $NF}'
done
cp _ab/new.so $L
