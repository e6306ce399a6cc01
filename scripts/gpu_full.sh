# full GPU suite + smoke + bench line
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err; tail -2 gpurun_out/bench_r02.err
python -c "
import json; d=json.load(open('gpurun_out/bench_r02.json'))
print('value', d['value']/1e9, 'C2', d['build']['ms'], d['build']['frac_of_hbm'])
for k,v in d['builds'].items(): print(k, round(v['ms'],3), round(v['ms_min'],3), round(v['frac_of_hbm'],3), round(v['ms_histogram_and_plan'],3))
"
