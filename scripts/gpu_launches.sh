set -x
mkdir -p gpurun_out
for d in 1 0; do
WT_DIR=$d timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_dir$d.csv python tools/bench_build.py --n-log 30 --sigma 256 --reps 0 > /dev/null 2>&1
python tools/profile_summary.py launches gpurun_out/launch_dir$d.csv > gpurun_out/launch_dir$d.txt 2>&1
done
WT_DIR=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_c4.csv python tools/bench_build.py --n-log 32 --kind dna --reps 0 > /dev/null 2>&1
python tools/profile_summary.py launches gpurun_out/launch_c4.csv > gpurun_out/launch_c4.txt 2>&1
cat gpurun_out/launch_dir1.txt gpurun_out/launch_dir0.txt gpurun_out/launch_c4.txt
