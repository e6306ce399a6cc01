#!/bin/bash
# build/var_<name>/libwt_b200.so with extra nvcc flags (A/B experiments; point
# WT_B200_LIB at it).  usage: scripts/build_variant.sh <name> "<-D flags>"
set -e
name=$1; shift
extra="$*"
root=$(cd "$(dirname "$0")/.." && pwd)
out=$root/build/var_$name
mkdir -p $out
cd $root/paper_2505_03372_b200/csrc
for f in wt_capi wt_wlevel wt_hist wt_query wt_bits wt_qlayout wt_ops; do
  nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xcompiler -O3 \
       --expt-relaxed-constexpr $extra -c $f.cu -o $out/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libwt_b200.so $out/*.o -ldl
echo built $out/libwt_b200.so
