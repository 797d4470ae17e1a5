timeout 300 python tools/stamps_fused.py c3 1
timeout 300 python tools/stamps_fused.py c3 32
