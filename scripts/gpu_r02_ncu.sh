# round-2 final ncu evidence: bench launch list + ncu --set full of every kernel
set -x
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_r02.csv python bench.py --steps 1 --warmup 1 \
  --extra-builds "" --c5-queries 0 --no-e2e --no-cpu > gpurun_out/ncu_launches_r02.out 2>&1
python tools/profile_summary.py launches gpurun_out/launches_r02.csv > gpurun_out/launches_r02.txt 2>&1
head -30 gpurun_out/launches_r02.txt
timeout 2700 ncu -f --set full --clock-control none --import-source on -o /tmp/prof_all \
  python tools/every_kernel.py > gpurun_out/ncu_all.out 2>&1
tail -3 gpurun_out/ncu_all.out
ncu -i /tmp/prof_all.ncu-rep --page raw --csv > /tmp/prof_all_raw.csv 2>/dev/null
python tools/ncu_all_summary.py /tmp/prof_all_raw.csv "" gpurun_out/ncu_all_r02.json > gpurun_out/ncu_all_r02.txt 2>&1
python tools/profile_summary.py report /tmp/prof_all.ncu-rep > gpurun_out/ncu_all_report_r02.txt 2>&1
for k in wlevel_kernel wpair_kernel; do python tools/ncu_regions.py /tmp/prof_all.ncu-rep $k paper_2505_03372_b200/csrc/wt_wlevel.cu > gpurun_out/regions_$k.txt 2>&1; done
python tools/ncu_regions.py /tmp/prof_all.ncu-rep dirq_kernel paper_2505_03372_b200/csrc/wt_qlayout.cu > gpurun_out/regions_dirq_kernel.txt 2>&1
head -50 gpurun_out/ncu_all_r02.txt
