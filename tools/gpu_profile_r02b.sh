#!/bin/bash
# Round-2 evidence capture (one gpurun call) for the current chain: launch lists of the bench command per config
# (cold, serialised), one `ncu --set full` per decode-step kernel at C3 / C2 / C4 (source-level), bench lines,
# smoke, timelines.   gpurun --timeout 2400 -- 'bash tools/gpu_profile_r02b.sh v2'
V=${1:-v2}
mkdir -p gpurun_out
for c in c3 c2 c4; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum \
    --clock-control none -k regex:"qq_kernel|select|token|attend" -s 8 -c 8 --csv --log-file gpurun_out/r02launch_${c}_${V}.csv \
    python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
for k in qq_kernel select_kernel token_pair_kernel attend_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^${k}" -s 3 -c 1 \
    -o gpurun_out/r02full_${k}_c3_${V} python tools/profile_step.py --config c3 --steps 3 > /dev/null 2>&1
done
for k in token_pair_kernel attend_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^${k}" -s 3 -c 1 \
    -o gpurun_out/r02full_${k}_c2_${V} python tools/profile_step.py --config c2 --steps 3 > /dev/null 2>&1
done
for k in token_pair_nt_kernel attend_mla_kernel select_kernel qq_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^${k}" -s 3 -c 1 \
    -o gpurun_out/r02full_${k}_c4_${V} python tools/profile_step.py --config c4 --steps 3 > /dev/null 2>&1
done
for c in c3 c2 c4; do
  timeout 600 python bench.py --config $c > gpurun_out/r02bench_${c}_${V}.json 2> gpurun_out/r02bench_${c}_${V}.err
done
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02smoke_${V}.log 2>&1
for c in c3 c2 c4; do timeout 200 python tools/timeline.py $c; done > gpurun_out/r02timeline_${V}.txt 2>&1
timeout 200 python tools/k2_stamps.py c3 > gpurun_out/r02k2stamps_${V}.txt 2>&1; timeout 200 python tools/k2_stamps.py c4 >> gpurun_out/r02k2stamps_${V}.txt 2>&1
ls gpurun_out/ | grep ${V} | wc -l
# summarise on the box (the .ncu-rep files exceed gpurun's 64 MiB return limit); keep the C3 token-kernel report
mkdir -p gpurun_out/prof_${V}
cp profiles/traffic.json gpurun_out/prof_${V}/traffic.json 2>/dev/null
TLS_PROFILES_OUT=gpurun_out/prof_${V} python tools/collect_r02.py ${V} > gpurun_out/prof_${V}/collect.log 2>&1
for f in gpurun_out/r02full_*_${V}.ncu-rep; do
  b=$(basename $f .ncu-rep)
  ncu -i $f --page source --csv --print-source=sass,cuda > gpurun_out/prof_${V}/${b}_source.csv 2>/dev/null
done
ls -la gpurun_out/prof_${V} | head -40
find gpurun_out -name "r02full_*_${V}.ncu-rep" ! -name "r02full_token_pair_kernel_c3_${V}.ncu-rep" -delete
du -sh gpurun_out
