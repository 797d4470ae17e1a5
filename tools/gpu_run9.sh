timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for c in c3 c2 c4; do timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], 'us/step', round(d['us_per_step'],1), 'e2e', round(d['e2e']['ms_per_step']*1e3,1), {k:round(v['avg_us'],1) for k,v in d['kernels'].items()}, d['roofline']['timing'])"; done
TLS_NO_PDL=1 timeout 300 python bench.py --config c3 --steps 200 --warmup 10 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('NO PDL', d['config']['workload'], 'us/step', round(d['us_per_step'],1))"
