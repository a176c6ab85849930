# Round-end style check on one B200: GPU tests, smoke, the default bench line,
# the reference arm, every config and every 8f row through bench.py, the scheme
# comparison, the inverse bench and the parity report (outputs: gpurun_out/).
set -x
mkdir -p gpurun_out/bench
timeout 2800 python -m pytest tests -m gpu -q -x 2>&1 | tail -4; [ ${PIPESTATUS[0]} -eq 0 ] || exit 1
timeout 120 python __graft_entry__.py smoke
timeout 600 python bench.py > gpurun_out/bench/default_c3.json 2> gpurun_out/bench/default_c3.err; tail -1 gpurun_out/bench/default_c3.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench/reference_c3.json 2>&1; tail -1 gpurun_out/bench/reference_c3.json
for c in 1 2 4 4b 5; do
  timeout 600 python bench.py --config $c > gpurun_out/bench/fwd53_c$c.json 2> gpurun_out/bench/fwd53_c$c.err
done
for c in 2 3 4 5; do timeout 600 python bench.py --config $c --op inverse > gpurun_out/bench/inv53_c$c.json 2>/dev/null; done
for c in 3 4; do
  timeout 600 python bench.py --config $c --wavelet cdf97 > gpurun_out/bench/fwd97_c$c.json 2>/dev/null
  timeout 600 python bench.py --config $c --wavelet cdf97 --op inverse > gpurun_out/bench/inv97_c$c.json 2>/dev/null
done
for sch in nonsep_naive nonsep_lifting nonsep_adapted sep_conv sep_lifting; do
  timeout 600 python bench.py --config 3 --scheme $sch > gpurun_out/bench/scheme_${sch}_c3.json 2>/dev/null
done
timeout 900 python scripts/scheme_compare.py > gpurun_out/scheme_compare.log 2>&1; tail -8 gpurun_out/scheme_compare.log
timeout 600 python scripts/inverse_bench.py > gpurun_out/inverse_bench.log 2>&1
timeout 1500 python tests/report_parity.py --out gpurun_out/parity_report.md > gpurun_out/parity_report.log 2>&1; tail -2 gpurun_out/parity_report.log
for f in gpurun_out/bench/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d.get('roofline') or {}
print('$f'.split('/')[-1], round(d['value'],2), d['unit'], 'ms', round(d['ms_per_step'],4), 'frac', round(r.get('frac',0),3), 'e2e', round(d['e2e']['value'],2) if d.get('e2e') else None, 'cpu', round(d['cpu_baseline']['value'],4) if d.get('cpu_baseline') else None)" 2>/dev/null || echo "$f: no line"; done
