# K = 2 warm-up peel on the register paths (forward + inverse), steady-state body as before:
# parity, base vs new of the 9/7 rows (-> gpurun_out/k2warm4/)
set -x
B=gpurun_out/k2warm4
mkdir -p $B
timeout 900 python -m pytest tests/test_gpu_wavelet97.py tests/test_gpu_fuzz.py tests/test_gpu_tail.py tests/test_gpu_small.py -q -x 2>&1 | tail -2
for c in 4 4b 3; do
for v in base new; do
  L=""; [ $v = base ] && L="--variant-lib build/variants/libdwt2_base.so"
  timeout 600 python bench.py $L --config $c --wavelet cdf97 --no-e2e --no-cpu-baseline > $B/f97_c${c}_${v}.json 2>/dev/null
  timeout 600 python bench.py $L --config $c --wavelet cdf97 --op inverse --no-e2e --no-cpu-baseline > $B/i97_c${c}_${v}.json 2>/dev/null
done
done
timeout 600 python bench.py --config 4 --wavelet cdf97 --no-e2e --no-cpu-baseline > $B/f97_c4_new2.json 2>/dev/null
timeout 600 python bench.py --variant-lib build/variants/libdwt2_base.so --config 4 --wavelet cdf97 --no-e2e --no-cpu-baseline > $B/f97_c4_base2.json 2>/dev/null
for f in $B/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d.get('roofline') or {}; st=d.get('step_stats') or {}; g=d.get('gate') or {}
print('$f'.split('/')[-1], round(d.get('value',0),2), 'ms', round(d.get('ms_per_step',0),4), 'med', st.get('median_ms'), 'frac', round(r.get('frac',0) or 0,3), 'gate', g.get('status'), 'clk', (d.get('clocks') or {}).get('reasons'))" 2>/dev/null || echo "$f: no line"; done
