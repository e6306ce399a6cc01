set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_large_gpu.py -x -q -k "block_mode or large_build" > gpurun_out/pytest_h.txt 2>&1; tail -3 gpurun_out/pytest_h.txt
for r in 1 2 4 8; do echo "== HREP $r"; WT_HREP=$r timeout 300 python tools/bench_build.py --n-log 30 --sigma 256 2>&1 | tail -2; done
for r in 1 4 8; do echo "== HREP $r dna"; WT_HREP=$r timeout 300 python tools/bench_build.py --n-log 32 --kind dna --reps 3 2>&1 | tail -1; done
