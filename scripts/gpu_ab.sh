# A/B of library variants on the build sweep: bash scripts/gpu_ab.sh lib1 lib2 ...
# (configs from $AB_CFGS, ';'-separated, default C2 and C3u)
set -x
IFS=';' read -ra CFGS <<< "${AB_CFGS:---n-log 30 --sigma 256;--n-log 30 --sigma 65536 --reps 3}"
for lib in "$@"; do echo "== $lib"; for a in "${CFGS[@]}"; do WT_B200_LIB=$lib timeout 300 python tools/bench_build.py $a 2>&1 | tail -1; done; done > gpurun_out/ab.txt 2>&1
cat gpurun_out/ab.txt
