set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"access_kernel|rank_kernel|select_kernel" -c 3 -o gpurun_out/prof_query3 python tools/bench_query.py --n-log 30 --sigma 256 --m 4000000 --reps 1 > gpurun_out/ncu_query3.out 2>&1
tail -3 gpurun_out/ncu_query3.out
