set -x
mkdir -p gpurun_out
rm -f gpurun_out/ab.txt
timeout 900 python -m pytest tests/test_large_gpu.py tests/test_parity_gpu.py -x -q > gpurun_out/pytest_large.txt 2>&1; tail -3 gpurun_out/pytest_large.txt
run() {  # label, env...
  local label=$1; shift
  echo "== $label" >> gpurun_out/ab.txt
  for a in "--n-log 30 --sigma 256" "--n-log 30 --sigma 65536 --reps 3" "--n-log 32 --kind dna --reps 3"; do
    env "$@" timeout 300 python tools/bench_build.py $a 2>&1 | tail -1 >> gpurun_out/ab.txt
  done
}
run dir WT_X=1
run nodir WT_DIR=0
run dir_again WT_X=1
cat gpurun_out/ab.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_dir.csv python tools/bench_build.py --n-log 30 --sigma 256 --reps 0 > /dev/null 2>&1
python tools/profile_summary.py launches gpurun_out/launch_dir.csv > gpurun_out/launch_dir.txt 2>&1; head -12 gpurun_out/launch_dir.txt
timeout 900 python -m pytest tests/test_configs_gpu.py -x -q > gpurun_out/pytest_cfg.txt 2>&1; tail -3 gpurun_out/pytest_cfg.txt
