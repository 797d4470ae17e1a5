#!/bin/bash
# A/B of an env knob on the bench (same box): bash tools/gpu_ab.sh <tag> "<ENV=val>" [configs]
T=${1:-ab}; ENVB=${2:-TLS_STREAM_SEL=0}; CFGS=${3:-c3 c2}
mkdir -p gpurun_out
for c in $CFGS; do
  for arm in A B A B; do
    if [ $arm = A ]; then E=""; else E="$ENVB"; fi
    env $E timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/${T}_$c_$arm.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/${T}_$c_$arm.json').read().strip().splitlines()[-1]); print('$c $arm', round(d['us_per_step'],1), {k: round(v['avg_us'],1) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])" 2>&1 | tail -1
  done
done
