# C2 build: launch list + ncu --set full of the pre-phase / directory / layout kernels
set -x
mkdir -p gpurun_out /tmp/prof
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/c2_launches.csv python tools/bench_build.py --n-log 30 --sigma 256 --reps 0 > /tmp/prof/l.out 2>&1
python tools/profile_summary.py launches gpurun_out/c2_launches.csv > gpurun_out/c2_launches.txt 2>&1
cat gpurun_out/c2_launches.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dir_kernel|qlayout_kernel|hist8_blocks|wpair|l1_scan|block_l1" -c 8 -o /tmp/prof/c2 python tools/bench_build.py --n-log 30 --sigma 256 --reps 0 > /tmp/prof/c2.out 2>&1
tail -3 /tmp/prof/c2.out
python tools/profile_summary.py report /tmp/prof/c2.ncu-rep > gpurun_out/sum_c2.txt 2>&1
for k in dir_kernel qlayout_kernel hist8_blocks_kernel; do python tools/ncu_lines.py /tmp/prof/c2.ncu-rep $k > gpurun_out/lines_$k.txt 2>&1; done
cp /tmp/prof/c2.ncu-rep gpurun_out/ 2>/dev/null
head -80 gpurun_out/sum_c2.txt
