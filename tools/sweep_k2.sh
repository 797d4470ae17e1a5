#!/bin/bash
# K2 chunking sweep: register-resident (default, nch 8) vs two-pass with larger chunks
b() { timeout 300 python bench.py --config ${1:-c3} --steps 100 --warmup 10 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json, sys; d = json.loads(sys.stdin.read())
print(d['config']['workload'], 'us/step', round(d['us_per_step'], 1), {k: round(v['avg_us'], 1) for k, v in d['kernels'].items()})"; }
for c in c3 c2; do
  echo "default"; b $c
  for cb in 16 32 64; do echo "two-pass cb=$cb"; TLS_K2_TWO_PASS=1 TLS_CHUNK_BLOCKS=$cb b $c; done
done
