M="gpu__time_duration.sum,dram__bytes_read.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size"
TLS_FUSED_MODE=1 timeout 300 ncu --metrics $M --clock-control none -k regex:"select|token|attend" -c 3 --csv --log-file gpurun_out/inst_m1.csv python tools/profile_step.py --config c3 --steps 1 > /dev/null 2>&1
timeout 300 ncu --metrics $M --clock-control none -k regex:"select|token|attend" -c 2 --csv --log-file gpurun_out/inst_m2.csv python tools/profile_step.py --config c3 --steps 1 > /dev/null 2>&1
