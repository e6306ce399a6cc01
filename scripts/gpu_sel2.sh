# A/B: sorted select walk, one vs two walks per thread (WT_SEL2)
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_large_gpu.py tests/test_parity_gpu.py -x -q -k "sort or select" > gpurun_out/pytest_sel.txt 2>&1; tail -2 gpurun_out/pytest_sel.txt
WT_SEL2=1 timeout 600 python -m pytest tests/test_large_gpu.py tests/test_parity_gpu.py -x -q -k "sort or select" > gpurun_out/pytest_sel2.txt 2>&1; tail -2 gpurun_out/pytest_sel2.txt
timeout 300 python tools/bench_query.py --sort 2>&1 | tail -4
WT_SEL2=1 timeout 300 python tools/bench_query.py --sort 2>&1 | tail -4
