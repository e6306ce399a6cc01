# PRMT pair kernel: parity first, then build timings (A/B against the staging pair)
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_large_gpu.py -k "pair or single_level or block_mode" -x -q > gpurun_out/pytest_pair.txt 2>&1; tail -15 gpurun_out/pytest_pair.txt
for pk in new stage; do
(for a in "--n-log 30 --sigma 256" "--n-log 30 --sigma 65536 --reps 3" "--n-log 32 --kind dna --reps 3"; do WT_PAIR_KERNEL=$pk timeout 300 python tools/bench_build.py $a 2>&1 | tail -1; done) > gpurun_out/pair2_build_$pk.txt 2>&1
cat gpurun_out/pair2_build_$pk.txt
done
timeout 1200 python -m pytest tests/test_configs_gpu.py tests/test_parity_gpu.py -x -q > gpurun_out/pytest_cfg.txt 2>&1; tail -5 gpurun_out/pytest_cfg.txt
