#!/bin/bash
b() { timeout 300 python bench.py --config ${1:-c4} --steps 100 --warmup 10 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json, sys; d = json.loads(sys.stdin.read())
print(d['config']['workload'], 'us/step', round(d['us_per_step'], 1), {k: round(v['avg_us'], 1) for k, v in d['kernels'].items()})"; }
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for kb in 32 64 96 128; do echo "tile=$kb KB"; TLS_TILE_KB=$kb b c4; done
b c3; b c2
