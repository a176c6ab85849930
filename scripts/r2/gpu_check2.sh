mkdir -p gpurun_out/r2h
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
for c in 4 4b 1 3; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/r2h/fwd53_c$c.json 2>gpurun_out/r2h/fwd53_c$c.err; python -c "import json; d=json.loads(open('gpurun_out/r2h/fwd53_c$c.json').read().strip().splitlines()[-1]); print('c$c', round(d['value'],1), round(d['ms_per_step']*1e3,2), d['gate']['status'], d['step_stats'].get('median_ms'), d['gpu_launches'])"; done
