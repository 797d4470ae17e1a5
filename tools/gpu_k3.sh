#!/bin/bash
# Attention iteration: sequence-split + parity tests, C3/C2 bench lines, C3 with two attention CTAs per pair.
mkdir -p gpurun_out
V=${1:-x}
timeout 900 python -m pytest tests/test_gpu_seqsplit.py tests/test_gpu_sanitizer.py tests/test_gpu_parity.py -x -q -k "not full_size and not budgets and not sanitizer" > gpurun_out/k3_tests_${V}.log 2>&1
tail -3 gpurun_out/k3_tests_${V}.log
for c in c3 c2; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --steps 300 --warmup 20 > gpurun_out/k3_bench_${c}_${V}.json 2> gpurun_out/k3_bench_${c}_${V}.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/k3_bench_${c}_${V}.json').read().strip().splitlines()[-1]); print('$c', round(d['ms_per_step']*1e3,1), 'us', {k: round(v['avg_us'],1) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])"
done
TLS_CLUSTER=2 timeout 300 python bench.py --config c3 --no-cpu-baseline --steps 300 --warmup 20 > gpurun_out/k3_bench_c3cs2_${V}.json 2>/dev/null
python -c "import json,sys; d=json.loads(open('gpurun_out/k3_bench_c3cs2_${V}.json').read().strip().splitlines()[-1]); print('c3 cs2', round(d['ms_per_step']*1e3,1), 'us', {k: round(v['avg_us'],1) for k,v in d['kernels'].items()})"
