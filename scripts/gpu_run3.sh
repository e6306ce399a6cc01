set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
WT_TRACE=1 timeout 300 python tools/bench_build.py --n-log 30 --sigma 256 --reps 6 2>&1 | tail -30
timeout 300 python tools/bench_query.py --n-log 30 --sigma 256
