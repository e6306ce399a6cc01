set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; tail -15 gpurun_out/pytest_gpu.txt
timeout 300 python tools/bench_query.py --n-log 30 --sigma 256 > gpurun_out/bench_query.txt 2>&1; cat gpurun_out/bench_query.txt
timeout 300 python tools/bench_query.py --n-log 30 --sigma 256 --sort > gpurun_out/bench_query_sort.txt 2>&1; cat gpurun_out/bench_query_sort.txt
