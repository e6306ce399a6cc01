# occupancy A/B of the level kernel: ring depth / min CTAs per SM (rebuilds wt_wlevel.o)
set -x
mkdir -p gpurun_out
BASE="-O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xcompiler -O3 -Xptxas -v --expt-relaxed-constexpr"
for v in "2 4 6" "1 6 6" "1 5 5" "2 5 6"; do
  set -- $v
  touch paper_2505_03372_b200/csrc/wt_wlevel.cu
  make -C paper_2505_03372_b200/csrc NVFLAGS="$BASE -DWT_W_RING=$1 -DWT_W_MINB4=$2 -DWT_W_MINB=$3" > /dev/null 2>&1
  echo "== ring $1 minb4 $2 minb $3" >> gpurun_out/occ.txt
  (for a in "--n-log 30 --sigma 256" "--n-log 30 --sigma 65536 --reps 3" "--n-log 32 --kind dna --reps 3"; do timeout 300 python tools/bench_build.py $a 2>&1 | tail -1; done) >> gpurun_out/occ.txt 2>&1
done
cat gpurun_out/occ.txt
