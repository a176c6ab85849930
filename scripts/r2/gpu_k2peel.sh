# Peeled warm-up on the K = 2 ring paths too, with fewer rows in flight (measurement builds
# under build/variants/; every line gated) -> gpurun_out/k2peel/
set -x
B=gpurun_out/k2peel
mkdir -p $B
V=build/variants
for c in 4 3; do
  for v in head2 fpeel_ds4 fpeel_ds3; do
    timeout 600 python bench.py --variant-lib $V/libdwt2_$v.so --config $c --wavelet cdf97 --no-e2e --no-cpu-baseline > $B/f97_c${c}_$v.json 2>/dev/null
  done
  for v in head2 ipeel ipeel_ds3; do
    timeout 600 python bench.py --variant-lib $V/libdwt2_$v.so --config $c --wavelet cdf97 --op inverse --no-e2e --no-cpu-baseline > $B/i97_c${c}_$v.json 2>/dev/null
  done
done
for f in $B/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d.get('roofline') or {}; st=d.get('step_stats') or {}; g=d.get('gate') or {}
print('$f'.split('/')[-1], round(d.get('value',0),2), 'ms', round(d.get('ms_per_step',0),4), 'med', st.get('median_ms'), 'frac', round(r.get('frac',0) or 0,3), 'gate', g.get('status'), 'clk', (d.get('clocks') or {}).get('reasons'))" 2>/dev/null || echo "$f: no line"; done
