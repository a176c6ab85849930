# bench.py over the non-default operations: inverse, the comparison schemes, CDF 9/7
mkdir -p gpurun_out/ops
one() { timeout 600 python bench.py "$@" 2>/dev/null | tail -1; }
for c in 3 4 2 5; do one --config $c --op inverse > gpurun_out/ops/inv_c$c.json; done
for sch in nonsep_naive nonsep_lifting nonsep_adapted sep_conv sep_lifting; do one --config 3 --scheme $sch > gpurun_out/ops/scheme_$sch.json; done
for c in 3 4; do one --config $c --wavelet cdf97 --op inverse > gpurun_out/ops/inv97_c$c.json; done
for f in gpurun_out/ops/*.json; do python -c "
import json,sys; d=json.loads(open('$f').read()); r=d['roofline']
print('$f'.split('/')[-1], round(d['value'],1), 'ms', round(d['ms_per_step'],4), 'frac', round(r['frac'],3), 'cpu', round(d['cpu_baseline']['value'],4) if d.get('cpu_baseline') else None, 'e2e', round(d['e2e']['value'],2) if d.get('e2e') else None)" || echo "$f failed"; done
