# HEAD bench lines of every config / 8f row (no cpu_baseline leg; the default line in
# last/default_c3.json carries it), the reference arm and the default launch list
# (-> gpurun_out/r2last/)
set -x
B=gpurun_out/r2last
mkdir -p $B
timeout 300 python bench.py --impl reference > $B/reference_c3.json 2>&1; tail -c 300 $B/reference_c3.json
for c in 1 2 4b 5; do timeout 300 python bench.py --config $c --no-cpu-baseline > $B/fwd53_c$c.json 2> $B/fwd53_c$c.err; done
for c in 2 3 4 4b 5; do timeout 300 python bench.py --config $c --op inverse --no-cpu-baseline > $B/inv53_c$c.json 2> $B/inv53_c$c.err; done
for c in 3 4 4b; do
  timeout 300 python bench.py --config $c --wavelet cdf97 --no-cpu-baseline > $B/fwd97_c$c.json 2> $B/fwd97_c$c.err
  timeout 300 python bench.py --config $c --wavelet cdf97 --op inverse --no-cpu-baseline > $B/inv97_c$c.json 2> $B/inv97_c$c.err
done
for f in $B/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d.get('roofline') or {}; st=d.get('step_stats') or {}; g=d.get('gate') or {}
print('$f'.split('/')[-1], round(d.get('value',0),2), d.get('unit'), 'ms', round(d.get('ms_per_step',0),4), 'med', st.get('median_ms'), 'frac', round(r.get('frac',0) or 0,3), 'gate', g.get('status'), 'e2e', round(d['e2e']['value'],2) if d.get('e2e') else None, 'clk', (d.get('clocks') or {}).get('reasons'))" 2>/dev/null || echo "$f: no line"; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $B/launches_default_c3.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-gate --stat-steps 2 > $B/ncu_default.log 2>&1
ls -la $B | tail -30
