# Last validation of HEAD this round: smoke, the GPU suite, default bench, 9/7 config 4b
# (-> gpurun_out/r2last/)
set -x
B=gpurun_out/r2last
mkdir -p $B
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python __graft_entry__.py smoke
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 600 python bench.py > $B/default_c3.json 2> $B/default_c3.err; tail -c 400 $B/default_c3.json
timeout 600 python bench.py --config 4 > $B/fwd53_c4.json 2> $B/fwd53_c4.err
for f in $B/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d.get('roofline') or {}; st=d.get('step_stats') or {}; g=d.get('gate') or {}
print('$f'.split('/')[-1], round(d.get('value',0),2), d.get('unit'), 'ms', round(d.get('ms_per_step',0),4), 'med', st.get('median_ms'), 'frac', round(r.get('frac',0) or 0,3), 'gate', g.get('status'), 'e2e', round(d['e2e']['value'],2) if d.get('e2e') else None, 'clk', (d.get('clocks') or {}).get('reasons'))" 2>/dev/null || echo "$f: no line"; done
ls -la $B
