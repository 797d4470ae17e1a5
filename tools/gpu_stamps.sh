mkdir -p gpurun_out
timeout 200 python tools/k2_stamps.py c3 > gpurun_out/k3stamps_c3.txt 2>&1
timeout 200 python tools/k2_stamps.py c4 >> gpurun_out/k3stamps_c3.txt 2>&1
cat gpurun_out/k3stamps_c3.txt
