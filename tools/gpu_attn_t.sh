#!/bin/bash
# tokens-as-M attention check: parity + bench with and without the heads-as-M fallback
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for v in "" 1; do
  export TLS_ATTN_HEADS_AS_M=$v; [ -z "$v" ] && unset TLS_ATTN_HEADS_AS_M
  timeout 200 python tools/attend_probe.py c3 2>&1 | tail -8
  for c in c3 c2; do
    timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json, sys; d = json.loads(sys.stdin.read())
print(d['config']['workload'], 'us/step', round(d['us_per_step'], 1), {k: round(v['avg_us'], 1) for k, v in d['kernels'].items()})"
  done
done
