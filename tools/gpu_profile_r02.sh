#!/bin/bash
# Round-2 evidence capture (one gpurun call): launch lists of the bench command per config (cold, serialised),
# one `ncu --set full` per decode-step kernel at C3 and C4 (source-level), bench lines, smoke.
#   gpurun --timeout 2400 -- 'bash tools/gpu_profile_r02.sh v1'
V=${1:-v1}
mkdir -p gpurun_out
for c in c3 c2 c4; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum \
    --clock-control none -k regex:"qq_kernel|select|token|attend" -s 8 -c 8 --csv --log-file gpurun_out/r02launch_${c}_${V}.csv \
    python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
for k in qq_kernel select_kernel token_reg_kernel attend_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^${k}" -s 3 -c 1 \
    -o gpurun_out/r02full_${k}_c3_${V} python tools/profile_step.py --config c3 --steps 3 > /dev/null 2>&1
done
for k in token_cluster_kernel attend_mla_kernel select_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^${k}" -s 3 -c 1 \
    -o gpurun_out/r02full_${k}_c4_${V} python tools/profile_step.py --config c4 --steps 3 > /dev/null 2>&1
done
for c in c3 c2 c4; do
  timeout 600 python bench.py --config $c > gpurun_out/r02bench_${c}_${V}.json 2> gpurun_out/r02bench_${c}_${V}.err
done
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02smoke_${V}.log 2>&1
for c in c3 c2 c4; do timeout 200 python tools/timeline.py $c; done > gpurun_out/r02timeline_${V}.txt 2>&1
ls gpurun_out/ | grep ${V} | wc -l
