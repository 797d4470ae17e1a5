#!/bin/bash
# Round check in one gpurun call: GPU tests (all), smoke, the driver's default bench line, C2/C4 bench lines.
#   bash tools/gpu_round.sh <tag>
T=${1:-r}
mkdir -p gpurun_out
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/${T}_gputests.log 2>&1; tail -3 gpurun_out/${T}_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; tail -1 gpurun_out/${T}_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${T}_bench_default.json 2> gpurun_out/${T}_bench_default.err
tail -c 1500 gpurun_out/${T}_bench_default.json
for c in c2 c4; do
  timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/${T}_bench_$c.json 2> gpurun_out/${T}_bench_$c.err
  python -c "
import json; d=json.loads(open('gpurun_out/${T}_bench_$c.json').read().strip().splitlines()[-1]); print('$c', round(d['us_per_step'],1), {k: round(v['avg_us'],1) for k,v in d['kernels'].items()}, d['clocks'])" 2>&1 | tail -1
done
