set -x
mkdir -p gpurun_out
(for a in "--n-log 30 --sigma 256" "--n-log 30 --sigma 65536 --reps 3" "--n-log 32 --kind dna --reps 3"; do echo "== $a"; timeout 300 python tools/bench_build.py $a 2>&1 | tail -2; done) > gpurun_out/pre_ab.txt 2>&1
cat gpurun_out/pre_ab.txt
WT_TRACE=1 python tools/bench_build.py --n-log 30 --sigma 256 --reps 1 2>&1 | tail -9
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_qlayout_gpu.py -x -q > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
