# pair mode: parity + build timings (A/B with WT_PAIR=0)
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_large_gpu.py -k "pair or single_level or block_mode" -x -q > gpurun_out/pytest_pair.txt 2>&1; tail -15 gpurun_out/pytest_pair.txt
for pe in 1 0; do
(for a in "--n-log 30 --sigma 256" "--n-log 30 --sigma 65536 --reps 3" "--n-log 32 --kind dna --reps 3"; do WT_PAIR=$pe timeout 300 python tools/bench_build.py $a 2>&1 | tail -2; done) > gpurun_out/pair_build_$pe.txt 2>&1
cat gpurun_out/pair_build_$pe.txt
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; tail -5 gpurun_out/pytest_gpu.txt
