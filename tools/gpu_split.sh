#!/bin/bash
mkdir -p gpurun_out
V=${1:-x}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "full_size or budgets or repeated or separate" > gpurun_out/split_tests_${V}.log 2>&1
tail -2 gpurun_out/split_tests_${V}.log
bash tools/gpu_ab.sh split "TLS_K3_SPLIT=0" "c3"
timeout 200 python tools/timeline.py c3 2>&1 | head -16
