# Round evidence: tests, smoke, bench (both arms), build sweep, launch list, ncu captures.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt
(nproc; lscpu | grep -E "Model name|^CPU\(s\)"; free -g) > gpurun_out/host.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -3 gpurun_out/bench_ref.err
(for a in "--n-log 30 --sigma 256" "--n-log 30 --sigma 65536" "--n-log 30 --kind zipf --sigma 65536 --declared --reps 3" "--n-log 32 --kind dna --reps 3"; do echo "== $a"; timeout 300 python tools/bench_build.py $a 2>&1 | tail -2; done) > gpurun_out/bench_build.txt 2>&1
timeout 300 python tools/bench_query.py --n-log 30 --sigma 256 > gpurun_out/bench_query.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --queries 30000000 --no-e2e --no-cpu > gpurun_out/ncu_launches.out 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wlevel_kernel -s 4 -c 1 -o gpurun_out/prof_level python tools/bench_build.py --n-log 30 --sigma 256 --reps 0 > gpurun_out/ncu_level.out 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"access_kernel|rank_kernel|select_kernel" -c 3 -o gpurun_out/prof_query python bench.py --steps 1 --warmup 0 --queries 3000000 --no-e2e --no-cpu --no-sort > gpurun_out/ncu_query.out 2>&1
ls -la gpurun_out
# the bench's own sorted batches (3.3e7 queries per kind): sort kernels, walks, gather
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"access_kernel|rank_kernel|select_kernel|qsort|qunsort" -c 21 -o gpurun_out/prof_query_sorted python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_query_sorted.out 2>&1
# dram traffic of the walk kernels at the bench's own batch size (feeds roofline.traffic)
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"access_kernel|rank_kernel|select_kernel" -c 3 --csv --log-file gpurun_out/traffic_full.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_traffic_full.out 2>&1
