set -x
mkdir -p gpurun_out /tmp/prof
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"wpair_kernel" -c 1 -o /tmp/prof/wl python tools/bench_build.py --n-log 30 --sigma 256 --reps 0 > /tmp/prof/wl.out 2>&1
tail -2 /tmp/prof/wl.out
python tools/profile_summary.py report /tmp/prof/wl.ncu-rep > gpurun_out/sum_wl.txt 2>&1
python tools/ncu_lines.py /tmp/prof/wl.ncu-rep wlevel_kernel > gpurun_out/lines_wl.txt 2>&1
python tools/ncu_lines.py /tmp/prof/wl.ncu-rep wpair_kernel > gpurun_out/lines_wp.txt 2>&1
python tools/ncu_regions.py /tmp/prof/wl.ncu-rep wlevel_kernel paper_2505_03372_b200/csrc/wt_wlevel.cu > gpurun_out/regions_wl.txt 2>&1
cp /tmp/prof/wl.ncu-rep gpurun_out/
grep -E "===|Duration|DRAM Through|Executed Inst|stall samples|Achieved Occ|Registers Per|Eligible|bank_conf|wavefronts_mem_shared" gpurun_out/sum_wl.txt; head -45 gpurun_out/lines_wl.txt; head -30 gpurun_out/regions_wl.txt
