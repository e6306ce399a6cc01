set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
bash scripts/gpu_ab.sh paper_2505_03372_b200/libwt_b200.so build/var/libwt_u8t2048.so
for lib in paper_2505_03372_b200/libwt_b200.so build/var/libwt_u8t2048.so; do WT_B200_LIB=$lib timeout 300 python tools/bench_build.py --n-log 32 --kind dna --reps 3 2>&1 | tail -1; done
