# round-2 evidence: tests, smoke, bench (both arms), build sweep, launch list, ncu of every kernel
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err; tail -3 gpurun_out/bench_r02.err
(for a in "--n-log 30 --sigma 256" "--n-log 30 --sigma 65536 --reps 3" "--n-log 30 --kind zipf --sigma 65536 --declared --reps 3" "--n-log 32 --kind dna --reps 3"; do echo "== $a"; timeout 300 python tools/bench_build.py $a 2>&1 | tail -2; done) > gpurun_out/bench_build_r02.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_r02.csv python bench.py --steps 1 --warmup 1 \
  --extra-builds "" --c5-queries 0 --no-e2e --no-cpu > gpurun_out/ncu_launches_r02.out 2>&1
python tools/profile_summary.py launches gpurun_out/launches_r02.csv > gpurun_out/launches_r02.txt 2>&1
timeout 2400 ncu -f --set full --clock-control none --import-source on -o /tmp/prof_all \
  python tools/every_kernel.py > gpurun_out/ncu_all.out 2>&1
tail -3 gpurun_out/ncu_all.out
ncu -i /tmp/prof_all.ncu-rep --page raw --csv > /tmp/prof_all_raw.csv 2>/dev/null
python tools/ncu_all_summary.py /tmp/prof_all_raw.csv > gpurun_out/ncu_all_r02.txt 2>&1
python tools/profile_summary.py report /tmp/prof_all.ncu-rep > gpurun_out/ncu_all_report_r02.txt 2>&1
for k in wlevel_kernel wpair_kernel dirq_kernel; do python tools/ncu_regions.py /tmp/prof_all.ncu-rep $k paper_2505_03372_b200/csrc/$( [ $k = dirq_kernel ] && echo wt_qlayout.cu || echo wt_wlevel.cu) > gpurun_out/regions_$k.txt 2>&1; done
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_r02.json 2> gpurun_out/bench_ref_r02.err; tail -2 gpurun_out/bench_ref_r02.err
ls -la gpurun_out
