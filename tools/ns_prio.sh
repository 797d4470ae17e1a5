for c in c3 c2 c4; do for ns in 1 2 4; do for po in 0 1; do
if [ $po = 1 ]; then export TLS_PRIO_ORDER=1; else unset TLS_PRIO_ORDER; fi
r=$(TLS_NSPLIT=$ns timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['us_per_step'],1))")
echo "$c ns=$ns prio_order=$po $r"
done; done; done
