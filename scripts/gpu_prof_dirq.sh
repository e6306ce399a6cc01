set -x
mkdir -p gpurun_out /tmp/prof
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"dirq" -s 2 -c 1 -o /tmp/prof/dirq python tools/bench_build.py --n-log 30 --sigma 256 --reps 0 > /tmp/prof/dirq.out 2>&1
python tools/profile_summary.py report /tmp/prof/dirq.ncu-rep > gpurun_out/sum_dirq.txt 2>&1
ncu -i /tmp/prof/dirq.ncu-rep --page details --csv > gpurun_out/det_dirq.csv 2>&1
python tools/ncu_lines.py /tmp/prof/dirq.ncu-rep dirq > gpurun_out/lines_dirq.txt 2>&1
head -50 gpurun_out/sum_dirq.txt
