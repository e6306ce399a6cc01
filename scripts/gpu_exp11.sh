set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
(for lib in paper_2505_03372_b200/libwt_b200.so build/var/libwt_s1_b8.so build/var/libwt_s2_b8.so build/var/libwt_s1_b6.so; do echo $lib; for a in "--n-log 30 --sigma 256" "--n-log 30 --sigma 65536 --reps 3"; do WT_B200_LIB=$lib timeout 300 python tools/bench_build.py $a 2>&1 | tail -1; done; done) > gpurun_out/exp11.txt 2>&1
cat gpurun_out/exp11.txt
