set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"level_kernel|count0|hist8|tile_scan" -s 9 -c 8 -o gpurun_out/prof_level4 python tools/bench_build.py --n-log 30 --sigma 256 --reps 0 > gpurun_out/ncu_level4.out 2>&1
tail -3 gpurun_out/ncu_level4.out
