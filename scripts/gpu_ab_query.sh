# A/B of library variants on the device query rates, sorted and unsorted:
# bash scripts/gpu_ab_query.sh lib1 lib2 ...
set -x
for lib in "$@"; do echo "== $lib"; WT_B200_LIB=$lib timeout 300 python tools/bench_query.py --sort 2>&1 | grep -E "Gq/s"; echo "-- unsorted"; WT_B200_LIB=$lib timeout 300 python tools/bench_query.py --reps 3 2>&1 | grep -E "Gq/s"; done > gpurun_out/abq.txt 2>&1
cat gpurun_out/abq.txt
