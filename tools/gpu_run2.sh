set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -25
TLS_FUSED_MODE=1 timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python tools/kernel_times.py c3 1,8,32
timeout 300 python tools/kernel_times.py c2 16
timeout 300 python tools/kernel_times.py c4 32
