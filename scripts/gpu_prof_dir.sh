set -x
mkdir -p gpurun_out /tmp/prof
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"dir_kernel" -s 2 -c 1 -o /tmp/prof/dir python tools/bench_build.py --n-log 30 --sigma 256 --reps 0 > /tmp/prof/dir.out 2>&1
python tools/profile_summary.py report /tmp/prof/dir.ncu-rep > gpurun_out/sum_dir.txt 2>&1
python tools/ncu_lines.py /tmp/prof/dir.ncu-rep dir_kernel > gpurun_out/lines_dir.txt 2>&1
ncu -i /tmp/prof/dir.ncu-rep --page details --csv > gpurun_out/det_dir.csv 2>&1
head -40 gpurun_out/sum_dir.txt; head -25 gpurun_out/lines_dir.txt
