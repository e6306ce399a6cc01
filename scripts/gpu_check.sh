# quick check: GPU tests + build sweep + device query rates
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
(for a in "--n-log 30 --sigma 256" "--n-log 30 --sigma 65536 --reps 3" "--n-log 32 --kind dna --reps 3"; do timeout 300 python tools/bench_build.py $a 2>&1 | tail -1; done) > gpurun_out/check_build.txt 2>&1
cat gpurun_out/check_build.txt
timeout 300 python tools/bench_query.py --n-log 30 --sigma 256 --sort > gpurun_out/check_query.txt 2>&1; cat gpurun_out/check_query.txt
