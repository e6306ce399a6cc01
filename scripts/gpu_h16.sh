set -x
timeout 900 python -m pytest tests/test_large_gpu.py tests/test_parity_gpu.py -x -q -k "u16 or hist or 65536 or zipf or declared" > gpurun_out/pytest_h16.txt 2>&1; tail -2 gpurun_out/pytest_h16.txt
for a in "--n-log 30 --sigma 65536 --reps 3" "--n-log 30 --kind zipf --sigma 65536 --declared --reps 3"; do timeout 300 python tools/bench_build.py $a 2>&1 | tail -1; done
