#!/bin/bash
V=${1:-x}; K=${2:-token_pair_kernel}; C=${3:-c3}
mkdir -p gpurun_out
bash tools/gpu_k2.sh $V
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^${K}" -s 3 -c 1 \
    -o gpurun_out/ncu_${K}_${C}_${V} python tools/profile_step.py --config $C --steps 3 > gpurun_out/ncu_${K}_${V}.log 2>&1
tail -2 gpurun_out/ncu_${K}_${V}.log
