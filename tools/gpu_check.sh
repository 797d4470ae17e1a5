#!/bin/bash
# One gpurun call: GPU tests (incl. slow full-size parity), smoke, quick bench lines.  bash tools/gpu_check.sh <tag> [pytest -k expr]
T=${1:-chk}
K=${2:-}
mkdir -p gpurun_out
python -m paper_2604_07815_b200.build > gpurun_out/build_${T}.log 2>&1
if [ -n "$K" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x -k "$K" > gpurun_out/gputests_${T}.log 2>&1
else
  timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputests_${T}.log 2>&1
fi
tail -3 gpurun_out/gputests_${T}.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${T}.log 2>&1; tail -1 gpurun_out/smoke_${T}.log
for c in c3 c2 c4; do
  timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_${c}_${T}.json 2> gpurun_out/bench_${c}_${T}.err
  python -c "
import json, sys; d = json.loads(open('gpurun_out/bench_${c}_${T}.json').read())
print(d['config']['workload'], 'us/step', round(d['us_per_step'], 1), {k: round(v['avg_us'], 1) for k, v in d['kernels'].items()}, d['clocks'])" 2>&1 | tail -1
done
