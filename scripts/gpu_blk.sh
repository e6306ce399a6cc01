# block-mode levels: A/B build sweep, then the GPU tests
set -x
mkdir -p gpurun_out
for bl in 1 0; do
(for a in "--n-log 30 --sigma 256" "--n-log 30 --sigma 65536 --reps 3" "--n-log 32 --kind dna --reps 3"; do WT_BLK_LEVELS=$bl timeout 300 python tools/bench_build.py $a 2>&1 | tail -2; done) > gpurun_out/blk_build_$bl.txt 2>&1
cat gpurun_out/blk_build_$bl.txt
done
timeout 900 python -m pytest tests/test_large_gpu.py -x -q > gpurun_out/pytest_large.txt 2>&1; tail -5 gpurun_out/pytest_large.txt
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; tail -5 gpurun_out/pytest_gpu.txt
