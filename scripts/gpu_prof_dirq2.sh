set -x
mkdir -p gpurun_out /tmp/prof
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"dirq_kernel|l1_scan" -s 2 -c 3 -o /tmp/prof/dq python tools/bench_build.py --n-log 30 --sigma 256 --reps 0 > /tmp/prof/dq.out 2>&1
tail -2 /tmp/prof/dq.out
python tools/profile_summary.py report /tmp/prof/dq.ncu-rep > gpurun_out/sum_dq.txt 2>&1
python tools/ncu_lines.py /tmp/prof/dq.ncu-rep dirq_kernel > gpurun_out/lines_dq.txt 2>&1
cp /tmp/prof/dq.ncu-rep gpurun_out/
cat gpurun_out/sum_dq.txt | head -120; head -40 gpurun_out/lines_dq.txt
