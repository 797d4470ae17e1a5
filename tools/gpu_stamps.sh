mkdir -p gpurun_out
for c in c3 c2 c4; do timeout 200 python tools/k2_stamps.py $c 2>&1 | tail -7; done
