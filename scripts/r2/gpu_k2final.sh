set -x
B=gpurun_out/r2final
mkdir -p $B
timeout 900 python -m pytest tests/test_gpu_wavelet97.py tests/test_gpu_tail.py tests/test_gpu_fuzz.py -q -x 2>&1 | tail -2
timeout 900 python bench.py --config 4 --wavelet cdf97 > $B/fwd97_c4.json 2> $B/fwd97_c4.err
timeout 900 python bench.py --config 4b --wavelet cdf97 > $B/fwd97_c4b.json 2> $B/fwd97_c4b.err
for f in fwd97_c4 fwd97_c4b; do python -c "
import json; d=json.loads(open('$B/$f.json').read().strip().splitlines()[-1]); r=d.get('roofline') or {}; st=d.get('step_stats') or {}; g=d.get('gate') or {}
print('$f', round(d.get('value',0),2), 'ms', round(d.get('ms_per_step',0),4), 'med', st.get('median_ms'), 'frac', round(r.get('frac',0) or 0,3), 'gate', g.get('status'), 'clk', (d.get('clocks') or {}).get('reasons'))"; done
