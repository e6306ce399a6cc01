set -x
mkdir -p gpurun_out
for lib in paper_2505_03372_b200/libwt_b200.so build/var/libwt_nt128.so; do
  WT_B200_LIB=$lib timeout 300 python tools/bench_build.py --n-log 30 --sigma 256 --reps 4 2>&1 | tail -2
done > gpurun_out/exp1.txt 2>&1
WT_TRACE=1 timeout 300 python tools/bench_build.py --n-log 30 --sigma 65536 --reps 3 > gpurun_out/exp1_trace.txt 2>&1
