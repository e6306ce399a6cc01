# A/B of the sort kernels' queries per thread (sorted batches only), 2 rounds
set -x
mkdir -p gpurun_out
for r in 1 2; do for lib in "$@"; do echo "== $lib"; WT_B200_LIB=$lib timeout 300 python tools/bench_query.py --sort 2>&1 | grep -E "Gq/s"; done; done > gpurun_out/abqs.txt 2>&1
cat gpurun_out/abqs.txt
