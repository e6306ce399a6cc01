set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 300 python tools/bench_query.py --n-log 30 --sigma 256 > gpurun_out/bench_query.txt 2>&1; cat gpurun_out/bench_query.txt
timeout 120 ./tools/gather_peak > gpurun_out/gather_peak.txt 2>&1; cat gpurun_out/gather_peak.txt
timeout 900 python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
