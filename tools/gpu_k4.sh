#!/bin/bash
# G > 8 token kernel iteration: tests, C4 bench (auto / cluster), K2 stamps at C4.
mkdir -p gpurun_out
V=${1:-x}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "nt_forms or small or sink or forms" > gpurun_out/k4_tests_${V}.log 2>&1
tail -3 gpurun_out/k4_tests_${V}.log
for f in auto cluster; do
  if [ $f = auto ]; then unset TLS_K2_FORM; else export TLS_K2_FORM=$f; fi
  timeout 300 python bench.py --config c4 --no-cpu-baseline --steps 300 --warmup 20 > gpurun_out/k4_bench_${f}_${V}.json 2> gpurun_out/k4_bench_${f}_${V}.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/k4_bench_${f}_${V}.json').read().strip().splitlines()[-1]); print('$f c4', round(d['ms_per_step']*1e3,1), 'us', {k: round(v['avg_us'],1) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])"
done
unset TLS_K2_FORM
timeout 200 python tools/timeline.py c4 > gpurun_out/k4_timeline_${V}.txt 2>&1; cat gpurun_out/k4_timeline_${V}.txt
