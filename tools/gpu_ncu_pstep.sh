#!/bin/bash
# one ncu --set full capture (source-level) of the persistent step kernel at C3.  bash tools/gpu_ncu_pstep.sh <tag> [config]
T=${1:-n}; C=${2:-c3}
mkdir -p gpurun_out
TLS_PSTEP=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:pstep -s 3 -c 1 \
  -o gpurun_out/${T}_pstep_${C} python tools/profile_step.py --config $C --steps 4 > gpurun_out/${T}_ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/${T}_ncu.log
