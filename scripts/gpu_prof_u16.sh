set -x
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:wlevel_kernel -s 6 -c 1 -o gpurun_out/prof_u16 python tools/bench_build.py --n-log 28 --sigma 65536 --reps 0 > gpurun_out/ncu_u16.out 2>&1
tail -2 gpurun_out/ncu_u16.out
