#!/bin/bash
# One `ncu --set full` capture (source-level) per decode-step kernel at one config; reports land in gpurun_out/.
#   gpurun --timeout 1800 -- 'bash tools/gpu_ncu_c3.sh TAG [config] [kernels...]'
V=${1:-x}; C=${2:-c3}; shift 2
KS=${@:-select_kernel token_reg_kernel attend_kernel}
mkdir -p gpurun_out
for k in $KS; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^${k}" -s 3 -c 1 \
    -o gpurun_out/full_${k}_${C}_${V} python tools/profile_step.py --config $C --steps 3 > gpurun_out/full_${k}_${C}_${V}.log 2>&1
done
ls -la gpurun_out | grep _${V}
