#!/bin/bash
# persistent step kernel check: hang probe, per-item timeline, bench lines, parity.  bash tools/gpu_pstep.sh <tag>
T=${1:-p}
mkdir -p gpurun_out
timeout 60 python tools/pstep_hang.py c3 > gpurun_out/${T}_hang.log 2>&1; echo "hang rc=$?"; tail -2 gpurun_out/${T}_hang.log
if grep -q "no hang" gpurun_out/${T}_hang.log; then
  for c in c3 c2; do timeout 120 python tools/pstep_timeline.py $c 2>&1 | tail -7; done > gpurun_out/${T}_tl.txt; cat gpurun_out/${T}_tl.txt
  for c in c3 c2; do
    TLS_PSTEP=1 timeout 300 python bench.py --config $c --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/${T}_bench_$c.json 2> gpurun_out/${T}_bench_$c.err
    python -c "
import json; d=json.loads(open('gpurun_out/${T}_bench_$c.json').read().strip().splitlines()[-1]); print('$c', round(d['us_per_step'],1), d['config'].get('select_mode'), d['clocks'])" 2>&1 | tail -1
  done
  timeout 900 python -m pytest tests/test_gpu_pstep.py -q -x ${PYTEST_K} > gpurun_out/${T}_tests.log 2>&1; tail -15 gpurun_out/${T}_tests.log
fi
