set -x
mkdir -p gpurun_out
rm -f gpurun_out/san.txt
for a in "--n-log 24 --sigma 256" "--n-log 24 --sigma 65536" "--n-log 26 --kind zipf --sigma 38158" "--n-log 26 --kind zipf --sigma 65536 --declared" "--n-log 26 --kind dna"; do
  echo "== $a" >> gpurun_out/san.txt
  timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python tools/bench_build.py $a --reps 0 >> gpurun_out/san.txt 2>&1
done
echo "== C3r full" >> gpurun_out/san.txt
timeout 1200 compute-sanitizer --tool memcheck --print-limit 5 python tools/bench_build.py --n-log 30 --kind zipf --sigma 38158 --reps 0 >> gpurun_out/san.txt 2>&1
grep -v "^rep\|^built" gpurun_out/san.txt | tail -40
