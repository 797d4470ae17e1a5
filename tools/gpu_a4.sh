#!/bin/bash
mkdir -p gpurun_out
V=${1:-x}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "small or forms or separate or repeated or lag or edge or ties or sink or full_size or block_scores or mla" > gpurun_out/a4_tests_${V}.log 2>&1
tail -2 gpurun_out/a4_tests_${V}.log
for c in c3 c2 c4; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --steps 300 --warmup 20 > gpurun_out/a4_bench_${c}_${V}.json 2> gpurun_out/a4_bench_${c}_${V}.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/a4_bench_${c}_${V}.json').read().strip().splitlines()[-1]); print('$c', round(d['ms_per_step']*1e3,1), 'us', {k: round(v['avg_us'],1) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])"
done
for c in c3 c2; do timeout 200 python tools/k2_stamps.py $c 2>&1 | grep -E "cycles|top-k_t"; done
