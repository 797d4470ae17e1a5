#!/bin/bash
# Auxiliary measurements with clock records on the current code: budget / pattern sweep, operator comparison,
# offload engine (token cache and asynchronous block cache).
mkdir -p gpurun_out
V=${1:-x}
timeout 900 python tools/budget_sweep.py c3,c2 > gpurun_out/aux_budget_${V}.jsonl 2> gpurun_out/aux_budget_${V}.err
timeout 900 python tools/compare_dense.py > gpurun_out/aux_compare_${V}.jsonl 2> gpurun_out/aux_compare_${V}.err
for b in 16 64; do timeout 600 python tools/offload_bench.py --batch $b --mode token >> gpurun_out/aux_offload_${V}.jsonl 2>> gpurun_out/aux_offload_${V}.err; done
timeout 600 python tools/offload_bench.py --batch 16 --mode block --layers 1 >> gpurun_out/aux_offload_${V}.jsonl 2>> gpurun_out/aux_offload_${V}.err
timeout 600 python tools/offload_bench.py --batch 16 --mode block --layers 4 >> gpurun_out/aux_offload_${V}.jsonl 2>> gpurun_out/aux_offload_${V}.err
timeout 900 python tools/offload_bench.py --batch 64 --mode block --layers 2 >> gpurun_out/aux_offload_${V}.jsonl 2>> gpurun_out/aux_offload_${V}.err
wc -l gpurun_out/aux_*_${V}.jsonl
