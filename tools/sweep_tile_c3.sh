for c in c3 c2; do for kb in 16 24 32 48 64; do
r=$(TLS_TILE_KB=$kb timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['us_per_step'],1), {k: round(v['avg_us'],1) for k,v in d['kernels'].items()})")
echo "$c tile_kb=$kb $r"
done; done
TLS_NO_PDL=1 python tools/stamps.py c3
