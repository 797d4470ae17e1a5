set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
for c in c3 c2 c4; do timeout 300 python bench.py --config $c --steps 300 --warmup 10 --no-cpu-baseline 2>&1 | tail -1; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 8 --csv --log-file gpurun_out/launches_c3.csv python bench.py --config c3 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_b.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 8 --csv --log-file gpurun_out/launches_c4.csv python bench.py --config c4 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_b4.log 2>&1
