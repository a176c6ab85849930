set -x
for i in 1 2; do
for v in product old; do
  if [ $v = old ]; then VL="--variant-lib build/variants/libdwt2_old.so"; else VL=""; fi
  for c in 5 4 1; do
    timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --no-gate $VL 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v c$c', round(d['value'],1), round(d['ms_per_step']*1e3,2), 'us', (d.get('step_stats') or {}).get('median_ms'))"
  done
done
done
