# Re-entry validation of HEAD: smoke, the GPU suite, default bench + reference arm,
# the odd-pitch configs the last change touched (-> gpurun_out/r2head/)
set -x
B=gpurun_out/r2head
mkdir -p $B
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python __graft_entry__.py smoke
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 900 python bench.py > $B/default_c3.json 2> $B/default_c3.err; tail -c 400 $B/default_c3.json
timeout 900 python bench.py --impl reference > $B/reference_c3.json 2>&1; tail -c 300 $B/reference_c3.json
for c in 4 4b 5 2; do timeout 900 python bench.py --config $c > $B/fwd53_c$c.json 2> $B/fwd53_c$c.err; done
for c in 4b 5; do timeout 900 python bench.py --config $c --op inverse > $B/inv53_c$c.json 2> $B/inv53_c$c.err; done
for f in $B/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d.get('roofline') or {}; st=d.get('step_stats') or {}; g=d.get('gate') or {}
print('$f'.split('/')[-1], round(d.get('value',0),2), d.get('unit'), 'ms', round(d.get('ms_per_step',0),4), 'med', st.get('median_ms'), 'frac', round(r.get('frac',0) or 0,3), 'gate', g.get('status'), 'e2e', round(d['e2e']['value'],2) if d.get('e2e') else None, 'clk', (d.get('clocks') or {}).get('reasons'))" 2>/dev/null || echo "$f: no line"; done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $B/launches_default_c3.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-gate --stat-steps 2 > $B/ncu_default.log 2>&1
ls -la $B
