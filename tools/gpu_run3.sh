set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -25
timeout 300 python tools/stamps_fused.py c3 1
timeout 300 python tools/stamps_fused.py c3 32
timeout 300 python tools/kernel_times.py c3 1,8,32
