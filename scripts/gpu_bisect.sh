set -x
mkdir -p gpurun_out
CUDA_LAUNCH_BLOCKING=1 timeout 600 python bench.py --steps 2 --warmup 3 --extra-builds "" --no-cpu > gpurun_out/bis1.json 2> gpurun_out/bis1.err; grep -v Assertion gpurun_out/bis1.err | tail -12
CUDA_LAUNCH_BLOCKING=1 timeout 600 python bench.py --steps 2 --warmup 3 --extra-builds C4 --no-e2e --c5-queries 0 --no-cpu > gpurun_out/bis2.json 2> gpurun_out/bis2.err; grep -v Assertion gpurun_out/bis2.err | tail -12
