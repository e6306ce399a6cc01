set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python tools/bench_build.py --n-log 30 --sigma 256
timeout 300 python tools/bench_build.py --n-log 30 --sigma 65536
timeout 300 python tools/bench_build.py --n-log 32 --kind dna --reps 3
