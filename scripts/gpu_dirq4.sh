set -x
mkdir -p gpurun_out /tmp/prof
timeout 600 python -m pytest tests/test_qlayout_gpu.py -x -q > gpurun_out/pytest_ql.txt 2>&1; tail -15 gpurun_out/pytest_ql.txt
(for a in "--n-log 30 --sigma 256" "--n-log 30 --sigma 65536 --reps 3" "--n-log 32 --kind dna --reps 3"; do echo "== $a"; timeout 300 python tools/bench_build.py $a 2>&1 | tail -2; WT_DIRQ=0 timeout 300 python tools/bench_build.py $a 2>&1 | tail -1; done) > gpurun_out/dirq_ab.txt 2>&1
cat gpurun_out/dirq_ab.txt
timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:"dirq_kernel" -s 2 -c 1 -o /tmp/prof/dq python tools/bench_build.py --n-log 30 --sigma 256 --reps 0 > /tmp/prof/dq.out 2>&1
python tools/profile_summary.py report /tmp/prof/dq.ncu-rep > gpurun_out/sum_dq.txt 2>&1
python tools/ncu_lines.py /tmp/prof/dq.ncu-rep dirq_kernel > gpurun_out/lines_dq.txt 2>&1
cp /tmp/prof/dq.ncu-rep gpurun_out/
cat gpurun_out/sum_dq.txt | head -40; head -30 gpurun_out/lines_dq.txt

