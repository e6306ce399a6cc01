set -x
mkdir -p gpurun_out
(for a in "--n-log 30 --sigma 256" "--n-log 30 --sigma 65536 --reps 3" "--n-log 32 --kind dna --reps 3"; do timeout 300 python tools/bench_build.py $a 2>&1 | tail -1; done) > gpurun_out/dir2_build.txt 2>&1
cat gpurun_out/dir2_build.txt
timeout 900 python -m pytest tests/test_large_gpu.py tests/test_parity_gpu.py -x -q > gpurun_out/pytest_large.txt 2>&1; tail -3 gpurun_out/pytest_large.txt
timeout 1200 python -m pytest tests/test_configs_gpu.py -x -q > gpurun_out/pytest_cfg.txt 2>&1; tail -3 gpurun_out/pytest_cfg.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -12 gpurun_out/bench.err
