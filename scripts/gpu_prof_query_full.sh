# full-size sorted query profile: launch list + one ncu --set full capture of
# each walk kernel (C2 tree, 33.3 M queries per kind)
set -x
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/qlaunch.csv python tools/bench_query.py --sort --reps 1 > /dev/null 2>&1
python tools/profile_summary.py launches gpurun_out/qlaunch.csv > gpurun_out/qlaunch.txt 2>&1; head -14 gpurun_out/qlaunch.txt
for k in access_kernel rank_kernel select_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/prof_$k python tools/bench_query.py --sort --reps 0 > gpurun_out/ncu_$k.out 2>&1
  tail -1 gpurun_out/ncu_$k.out
done
