timeout 300 python tools/kernel_times.py c3 1,32
TLS_FUSED_MODE=1 timeout 300 python tools/kernel_times.py c3 1,32
TLS_FUSED_MODE=1 timeout 300 python tools/kernel_times.py c2 16
timeout 300 python tools/kernel_times.py c4 1,32
