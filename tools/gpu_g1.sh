mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt
for c in c3 c2; do timeout 120 python tools/pstep_hang.py $c > gpurun_out/g1_hang_$c.log 2>&1; echo "hang $c rc=$?"; tail -3 gpurun_out/g1_hang_$c.log; done
for c in c3 c2 c4; do
  timeout 300 python bench.py --config $c --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/g1_bench_$c.json 2> gpurun_out/g1_bench_$c.err; echo "bench $c rc=$?"
  TLS_NO_PSTEP=1 timeout 300 python bench.py --config $c --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/g1_bench_${c}_chain.json 2> gpurun_out/g1_bench_${c}_chain.err
done
for f in gpurun_out/g1_bench_*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['us_per_step'],1), d.get('config',{}).get('select_mode'), {k: round(v['avg_us'],1) for k,v in d['kernels'].items()}, d['clocks'])" 2>&1 | tail -1; done
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/g1_gputests.log 2>&1; tail -5 gpurun_out/g1_gputests.log
