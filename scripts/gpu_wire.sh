# narrow-wire e2e A/B + the parity tests that cover it
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/wire_pytest.txt 2>&1; tail -3 gpurun_out/wire_pytest.txt
for cfg in "1 16" "0 16" "1 8" "1 12"; do set -- $cfg; WT_WIRE=$1 WT_HOST_THREADS=$2 timeout 600 python bench.py --no-cpu --extra-builds "" --c5-queries 0 > gpurun_out/wire_$1_$2.json 2> gpurun_out/wire_$1_$2.err; python -c "
import json,sys; d=json.load(open('gpurun_out/wire_$1_$2.json')); e=d['e2e']; print('WT_WIRE=$1 threads $2 value', d['value']/1e9, 'e2e', e['value']/1e9, 'h2d', e['h2d_bytes_per_step'], e.get('narrow_chunks'), {k:round(v['ms'],2) for k,v in e['per_kind'].items()})" >> gpurun_out/wire_summary.txt; done
cat gpurun_out/wire_summary.txt
