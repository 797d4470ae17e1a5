#!/bin/bash
# GPU tests (-x) then bench lines for the given configs (default c3 c2 c3 c2): step time and serialised kernel times.
#   gpurun --timeout 1800 -- 'bash tools/gpu_check_bench.sh TAG [configs...]'
V=${1:-x}; shift
CS=${@:-c3 c2 c3 c2}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/tests_${V}.log 2>&1; tail -3 gpurun_out/tests_${V}.log
for c in $CS; do timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['config']['workload'], round(d['us_per_step'],1), {k: round(v['avg_us'],1) for k,v in d['kernels'].items()})"; done
