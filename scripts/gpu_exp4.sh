set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
(for lib in paper_2505_03372_b200/libwt_b200.so build/var/libwt_r3.so; do echo $lib; for a in "--n-log 30 --sigma 256" "--n-log 30 --sigma 65536" "--n-log 32 --kind dna --reps 3"; do WT_B200_LIB=$lib timeout 300 python tools/bench_build.py $a 2>&1 | tail -1; done; done) > gpurun_out/exp4.txt 2>&1
cat gpurun_out/exp4.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:wlevel_kernel -s 4 -c 1 -o gpurun_out/prof_wlevel3 python tools/bench_build.py --n-log 30 --sigma 256 --reps 0 > gpurun_out/ncu_wlevel3.out 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:wlevel_kernel -s 6 -c 1 -o gpurun_out/prof_wlevel3_u16 python tools/bench_build.py --n-log 28 --sigma 65536 --reps 0 > gpurun_out/ncu_wlevel3u16.out 2>&1
tail -2 gpurun_out/ncu_wlevel3.out
