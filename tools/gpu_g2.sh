mkdir -p gpurun_out
for L in "" "4,6,8" "8,12,14" "32,40,44"; do echo "== lags $L"; timeout 120 python tools/pstep_timeline.py c3 $L 2>&1 | tail -8; done > gpurun_out/g2_tl.txt
