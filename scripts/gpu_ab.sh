# A/B build timings: default library vs build/var_* variants, WT_DIR on/off
set -x
mkdir -p gpurun_out
run() {  # label, env...
  local label=$1; shift
  echo "== $label" >> gpurun_out/ab.txt
  for a in "--n-log 30 --sigma 256" "--n-log 30 --sigma 65536 --reps 3" "--n-log 32 --kind dna --reps 3"; do
    env "$@" timeout 300 python tools/bench_build.py $a 2>&1 | tail -1 >> gpurun_out/ab.txt
  done
}
run base WT_X=1
run scan2 WT_B200_LIB=build/var_scan2/libwt_b200.so
run base_nodir WT_DIR=0
run base_again WT_X=1
run pairstage WT_PAIR_KERNEL=stage
cat gpurun_out/ab.txt
timeout 900 python -m pytest tests/test_large_gpu.py -k "pair or block" -x -q > gpurun_out/pytest_pair.txt 2>&1; tail -3 gpurun_out/pytest_pair.txt
