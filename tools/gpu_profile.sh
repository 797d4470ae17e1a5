#!/bin/bash
# Committed-evidence capture (one gpurun call): launch list of the bench command
# (cold, serialised per-launch times), one `ncu --set full` capture per decode-step
# kernel at C3, and the bench lines.  Outputs land in gpurun_out/; summaries are
# copied to profiles/ by hand.  Run:  gpurun --timeout 2400 -- 'bash tools/gpu_profile.sh'
V=${1:-v15}
mkdir -p gpurun_out
for c in c3 c2 c4; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum \
    --clock-control none -k regex:"qq_kernel|select|token|attend" -s 8 -c 8 --csv --log-file gpurun_out/launches_${c}_${V}.csv \
    python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
for k in select_kernel token_reg_kernel attend_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
    -o gpurun_out/full_${k}_c3_${V} python tools/profile_step.py --config c3 --steps 3 > /dev/null 2>&1
done
for k in token_cluster_kernel attend_mla_kernel select_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
    -o gpurun_out/full_${k}_c4_${V} python tools/profile_step.py --config c4 --steps 3 > /dev/null 2>&1
done
for c in c3 c2 c4; do timeout 200 python tools/timeline.py $c; done > gpurun_out/timeline_${V}.txt 2>&1
for c in c3 c2 c4; do
  timeout 600 python bench.py --config $c > gpurun_out/bench_${c}_${V}.json 2> gpurun_out/bench_${c}_${V}.err
done
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${V}.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_${V}.json 2> gpurun_out/bench_ref_${V}.err
