set -x
nproc; free -g | head -2
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err
tail -3 gpurun_out/bench1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches1.csv python bench.py --steps 1 --warmup 1 --queries 30000000 --no-e2e --no-cpu > gpurun_out/ncu_bench1.out 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:level_kernel -s 3 -c 1 -o gpurun_out/prof_level python bench.py --steps 1 --warmup 0 --queries 3000000 --no-e2e --no-cpu > gpurun_out/ncu_level.out 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"select_kernel|rank_kernel|access_kernel" -c 3 -o gpurun_out/prof_query python bench.py --steps 1 --warmup 0 --queries 3000000 --no-e2e --no-cpu > gpurun_out/ncu_query.out 2>&1
ls -la gpurun_out
