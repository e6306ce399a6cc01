set -x
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err; grep -v Assertion gpurun_out/bench_r02.err | tail -5
timeout 900 python bench.py > gpurun_out/bench_r02b.json 2> gpurun_out/bench_r02b.err; grep -v Assertion gpurun_out/bench_r02b.err | tail -5
timeout 900 python -m pytest tests/test_large_gpu.py tests/test_configs_gpu.py -x -q > gpurun_out/pytest_lc.txt 2>&1; tail -3 gpurun_out/pytest_lc.txt
