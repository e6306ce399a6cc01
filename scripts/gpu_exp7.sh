set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
(for a in "--n-log 30 --sigma 256" "--n-log 30 --sigma 65536" "--n-log 32 --kind dna --reps 3"; do timeout 300 python tools/bench_build.py $a 2>&1 | tail -1; done) > gpurun_out/exp7.txt 2>&1; cat gpurun_out/exp7.txt
timeout 120 ./tools/gather_peak > gpurun_out/gather_peak.txt 2>&1; cat gpurun_out/gather_peak.txt
timeout 900 python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
