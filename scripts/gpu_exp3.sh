set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; tail -30 gpurun_out/pytest_gpu.txt
(for a in "--n-log 30 --sigma 256" "--n-log 30 --sigma 65536" "--n-log 32 --kind dna --reps 3"; do timeout 300 python tools/bench_build.py $a 2>&1 | tail -2; done) > gpurun_out/exp3.txt 2>&1
cat gpurun_out/exp3.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:wlevel_kernel -s 4 -c 1 -o gpurun_out/prof_wlevel2 python tools/bench_build.py --n-log 30 --sigma 256 --reps 0 > gpurun_out/ncu_wlevel2.out 2>&1
tail -2 gpurun_out/ncu_wlevel2.out
