# round-2 baseline on one B200: GPU tests, default bench line, build sweep
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; tail -5 gpurun_out/pytest_gpu.txt
timeout 600 python bench.py > gpurun_out/bench.txt 2>&1; tail -2 gpurun_out/bench.txt
(for a in "--n-log 30 --sigma 256" "--n-log 30 --sigma 65536 --reps 3" "--n-log 32 --kind dna --reps 3"; do timeout 300 python tools/bench_build.py $a 2>&1 | tail -1; done) > gpurun_out/check_build.txt 2>&1
cat gpurun_out/check_build.txt
