set -x
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:wlevel_kernel -s 1 -c 1 -o gpurun_out/prof_shallow python tools/bench_build.py --n-log 30 --sigma 65536 --reps 0 > gpurun_out/ncu_deep.out 2>&1
tail -2 gpurun_out/ncu_deep.out
