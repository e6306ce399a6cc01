# A/B of build variants (build/var_*): device build times
set -x
for v in "" wp4 dq2 t2k; do
  echo "== variant ${v:-default}"
  if [ -n "$v" ]; then export WT_B200_LIB=$PWD/build/var_$v/libwt_b200.so; else unset WT_B200_LIB; fi
  for a in "--n-log 30 --sigma 256" "--n-log 32 --kind dna --reps 3"; do
    timeout 300 python tools/bench_build.py $a 2>&1 | tail -1
  done
done
