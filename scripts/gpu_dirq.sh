# fused directory + query-layout pass: layout tests, full GPU suite, C2/C3u/C4 build A/B (WT_DIRQ=0 = split path)
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_qlayout_gpu.py -x -q > gpurun_out/pytest_ql.txt 2>&1; tail -15 gpurun_out/pytest_ql.txt
(for a in "--n-log 30 --sigma 256" "--n-log 30 --sigma 65536 --reps 3" "--n-log 32 --kind dna --reps 3"; do echo "== $a"; timeout 300 python tools/bench_build.py $a 2>&1 | tail -2; WT_DIRQ=0 timeout 300 python tools/bench_build.py $a 2>&1 | tail -1; done) > gpurun_out/dirq_ab.txt 2>&1
cat gpurun_out/dirq_ab.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; tail -5 gpurun_out/pytest_gpu.txt
