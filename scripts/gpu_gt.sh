set -x
timeout 900 python -m pytest tests/test_large_gpu.py tests/test_parity_gpu.py tests/test_qlayout_gpu.py -x -q > gpurun_out/pytest_gt.txt 2>&1; tail -2 gpurun_out/pytest_gt.txt
for v in "" gt8; do
  echo "== variant ${v:-default}"
  if [ -n "$v" ]; then export WT_B200_LIB=$PWD/build/var_$v/libwt_b200.so; else unset WT_B200_LIB; fi
  for a in "--n-log 30 --sigma 256" "--n-log 30 --sigma 65536 --reps 3" "--n-log 30 --kind zipf --sigma 65536 --declared --reps 3" "--n-log 32 --kind dna --reps 3"; do
    timeout 300 python tools/bench_build.py $a 2>&1 | tail -1
  done
done
