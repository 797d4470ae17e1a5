#!/bin/bash
# Final evidence for a round (one gpurun call): GPU tests, smoke, bench lines (C3/C2/C4 + reference arm),
# launch lists and the step timeline.  bash tools/gpu_final.sh <V>
V=${1:-v18}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gputests_${V}.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${V}.log 2>&1
for c in c3 c2 c4; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum \
    --clock-control none -k regex:"qq_kernel|select|token|attend" -s 8 -c 8 --csv --log-file gpurun_out/launches_${c}_${V}.csv \
    python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
for c in c3 c2 c4; do timeout 200 python tools/timeline.py $c; done > gpurun_out/timeline_${V}.txt 2>&1
for c in c3 c2 c4; do
  timeout 600 python bench.py --config $c > gpurun_out/bench_${c}_${V}.json 2> gpurun_out/bench_${c}_${V}.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_${V}.json 2> gpurun_out/bench_ref_${V}.err
