#!/bin/bash
# One gpurun call's worth of diagnostics (run from the repo root on the GPU box):
#   gpurun --timeout 1500 -- 'bash tools/gpu_diag.sh > gpurun_out/diag.log 2>&1'
# GPU parity tests, one bench line per BASELINE.json config (summarised), live
# per-kernel times and the selection worker timeline.  Nothing here is a bench value
# except the bench.py lines.
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for c in c3 c2 c4; do
  timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json, sys; d = json.loads(sys.stdin.read())
print(d['config']['workload'], 'us/step', round(d['us_per_step'], 1), 'e2e us', round(d['e2e']['ms_per_step'] * 1e3, 1),
      {k: round(v['avg_us'], 1) for k, v in d['kernels'].items()})"
done
timeout 300 python tools/kernel_times.py c3 1,8,32
timeout 300 python tools/stamps_fused.py c3
