#!/bin/bash
b() { timeout 300 python bench.py --config ${1:-c4} --steps 100 --warmup 10 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json, sys; d = json.loads(sys.stdin.read())
print(d['config']['workload'], 'us/step', round(d['us_per_step'], 1), {k: round(v['avg_us'], 1) for k, v in d['kernels'].items()})"; }
for cs in 2 4 8; do echo "cs=$cs"; TLS_CLUSTER=$cs b c4; done
