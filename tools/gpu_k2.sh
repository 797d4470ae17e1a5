#!/bin/bash
# Token-kernel iteration: form tests + small parity + sinks, then C3/C2 bench lines per form and K2 phase stamps.
mkdir -p gpurun_out
V=${1:-x}
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "forms or small or sink or separate or repeated or lag or edge" > gpurun_out/k2_tests_${V}.log 2>&1
tail -3 gpurun_out/k2_tests_${V}.log
for f in auto 1 cluster; do
for c in c3 c2; do
  if [ $f = auto ]; then unset TLS_K2_FORM; else export TLS_K2_FORM=$f; fi
  timeout 300 python bench.py --config $c --no-cpu-baseline --steps 300 --warmup 20 > gpurun_out/k2_bench_${c}_${f}_${V}.json 2> gpurun_out/k2_bench_${c}_${f}_${V}.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/k2_bench_${c}_${f}_${V}.json').read().strip().splitlines()[-1]); print('$f $c', round(d['ms_per_step']*1e3,1), 'us', {k: round(v['avg_us'],1) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])"
done; done
unset TLS_K2_FORM
timeout 120 python tools/k2_stamps.py c3 > gpurun_out/k2_stamps_${V}.txt 2>&1
timeout 120 python tools/timeline.py c3 >> gpurun_out/k2_stamps_${V}.txt 2>&1
cat gpurun_out/k2_stamps_${V}.txt
