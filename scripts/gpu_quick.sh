# quick GPU check: parity tests, device query throughput (sorted and unsorted)
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 300 python tools/bench_query.py --n-log 30 --sigma 256 --sort > gpurun_out/bench_query.txt 2>&1; cat gpurun_out/bench_query.txt
timeout 300 python tools/bench_query.py --n-log 30 --sigma 256 > gpurun_out/bench_query_unsorted.txt 2>&1; cat gpurun_out/bench_query_unsorted.txt
