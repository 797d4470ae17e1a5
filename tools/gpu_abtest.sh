#!/bin/bash
# A/B of two builds (abA = base, abB = candidate): parity tests on B, then the bench on both.
mkdir -p gpurun_out
cp abB/libtls.so paper_2604_07815_b200/libtls.so
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "${1:-small or forms or full_size or budgets or sink or ties or empty}" > gpurun_out/abtest.log 2>&1
tail -3 gpurun_out/abtest.log
bash tools/ab.sh abA abB "${2:-c3 c2}"
cp abB/libtls.so paper_2604_07815_b200/libtls.so
