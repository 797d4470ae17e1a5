#!/bin/bash
# A/B of two library builds on the same box: bash tools/ab.sh <dirA> <dirB> [configs]
b() { timeout 300 python bench.py --config $1 --steps 200 --warmup 10 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json, sys; d = json.loads(sys.stdin.read())
print(d['config']['workload'], 'us/step', round(d['us_per_step'], 1), {k: round(v['avg_us'], 1) for k, v in d['kernels'].items()})"; }
for rep in 1 2; do for c in ${3:-c3 c2 c4}; do
  for v in $1 $2; do cp $v/libtls.so paper_2604_07815_b200/libtls.so; echo -n "$v "; b $c; done
done; done
