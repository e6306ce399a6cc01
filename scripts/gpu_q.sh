set -x
mkdir -p gpurun_out /tmp/prof
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_large_gpu.py -x -q > gpurun_out/pytest_q.txt 2>&1; tail -3 gpurun_out/pytest_q.txt
for qpt in 2 1; do
  WT_QPT=$qpt timeout 300 python tools/bench_query.py --n-log 30 --sigma 256 > gpurun_out/bq_uns_$qpt.txt 2>&1; tail -4 gpurun_out/bq_uns_$qpt.txt
done
timeout 300 python tools/bench_query.py --n-log 30 --sigma 256 --sort > gpurun_out/bq_sort.txt 2>&1; tail -4 gpurun_out/bq_sort.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"dir_kernel" -s 2 -c 1 -o /tmp/prof/dir python tools/bench_build.py --n-log 30 --sigma 256 --reps 0 > /tmp/prof/dir.out 2>&1
python tools/profile_summary.py report /tmp/prof/dir.ncu-rep > gpurun_out/sum_dir.txt 2>&1
python tools/ncu_lines.py /tmp/prof/dir.ncu-rep dir_kernel > gpurun_out/lines_dir.txt 2>&1
head -40 gpurun_out/sum_dir.txt; head -16 gpurun_out/lines_dir.txt
