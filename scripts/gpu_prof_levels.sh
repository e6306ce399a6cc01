# ncu --set full of the level kernels, summarised on the box (reports stay there)
set -x
mkdir -p gpurun_out /tmp/prof
cap() {  # name, kernel regex, skip, count, command...
  local name=$1 re=$2 skip=$3 cnt=$4; shift 4
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$re" -s $skip -c $cnt -o /tmp/prof/$name "$@" > /tmp/prof/$name.out 2>&1
  python tools/profile_summary.py report /tmp/prof/$name.ncu-rep > gpurun_out/sum_$name.txt 2>&1
  python tools/ncu_regions.py /tmp/prof/$name.ncu-rep "$re" paper_2505_03372_b200/csrc/wt_wlevel.cu > gpurun_out/reg_$name.txt 2>&1
}
cap l3 wlevel_kernel 3 1 python tools/bench_build.py --n-log 30 --sigma 256 --reps 0
cap l6 wlevel_kernel 6 1 python tools/bench_build.py --n-log 30 --sigma 256 --reps 0
cap c4 wlevel_kernel 0 1 python tools/bench_build.py --n-log 32 --kind dna --reps 0
cap u16l3 wlevel_kernel 3 1 python tools/bench_build.py --n-log 30 --sigma 65536 --reps 0
cap misc "hist8|dir_kernel|qlayout" 0 3 python tools/bench_build.py --n-log 30 --sigma 256 --reps 0
ls -la gpurun_out
