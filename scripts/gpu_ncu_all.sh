#!/bin/bash
# ncu evidence for every kernel: one full-set capture of tools/every_kernel.py
# (rendered to CSV pages on the box; the .ncu-rep is kept only if small),
# plus the launch list (device-time shares) of one bench step.
set -x
mkdir -p gpurun_out
timeout 2400 ncu --set full --clock-control none --import-source on -o /tmp/prof_all \
  python tools/every_kernel.py > gpurun_out/ncu_all.out 2>&1
tail -3 gpurun_out/ncu_all.out
ncu -i /tmp/prof_all.ncu-rep --page raw --csv > gpurun_out/prof_all_raw.csv 2>/dev/null
ncu -i /tmp/prof_all.ncu-rep --page details --csv > gpurun_out/prof_all_details.csv 2>/dev/null
ls -la /tmp/prof_all.ncu-rep
[ $(stat -c %s /tmp/prof_all.ncu-rep) -lt 40000000 ] && cp /tmp/prof_all.ncu-rep gpurun_out/
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_r02.csv python bench.py --steps 1 --warmup 1 \
  --extra-builds "" --c5-queries 0 --no-e2e --no-cpu > gpurun_out/ncu_launches_r02.out 2>&1
tail -2 gpurun_out/ncu_launches_r02.out
ls -la gpurun_out
