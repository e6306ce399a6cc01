set -x
mkdir -p gpurun_out /tmp/prof
timeout 600 python -m pytest tests/test_qlayout_gpu.py tests/test_parity_gpu.py -x -q > gpurun_out/pytest_ql.txt 2>&1; tail -3 gpurun_out/pytest_ql.txt
(for a in "--n-log 30 --sigma 256" "--n-log 30 --sigma 65536 --reps 3"; do echo "== $a"; timeout 300 python tools/bench_build.py $a 2>&1 | tail -2; done) > gpurun_out/dq5.txt 2>&1
cat gpurun_out/dq5.txt
timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:"dirq_kernel" -s 2 -c 1 -o /tmp/prof/dq python tools/bench_build.py --n-log 30 --sigma 256 --reps 0 > /tmp/prof/dq.out 2>&1
python tools/profile_summary.py report /tmp/prof/dq.ncu-rep > gpurun_out/sum_dq.txt 2>&1
python tools/ncu_lines.py /tmp/prof/dq.ncu-rep dirq_kernel > gpurun_out/lines_dq.txt 2>&1
cp /tmp/prof/dq.ncu-rep gpurun_out/
grep -E "Duration|DRAM Through|Executed Inst|stall samples|Achieved Occ" gpurun_out/sum_dq.txt; head -24 gpurun_out/lines_dq.txt
