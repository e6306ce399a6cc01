set -x
mkdir -p gpurun_out
for d in 1 0; do
(for a in "--n-log 30 --sigma 256" "--n-log 30 --sigma 65536 --reps 3"; do WT_DIR=$d timeout 300 python tools/bench_build.py $a 2>&1 | tail -1; done) > gpurun_out/dir_build_$d.txt 2>&1
cat gpurun_out/dir_build_$d.txt
done
timeout 900 python -m pytest tests/test_large_gpu.py -x -q > gpurun_out/pytest_large.txt 2>&1; tail -3 gpurun_out/pytest_large.txt
timeout 1200 python -m pytest tests/test_configs_gpu.py tests/test_parity_gpu.py -x -q > gpurun_out/pytest_cfg.txt 2>&1; tail -3 gpurun_out/pytest_cfg.txt
