set -x
mkdir -p gpurun_out
timeout 900 python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
