mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_wavelet97.py -q -x 2>&1 | tail -15
for c in 3 2 4 5; do
  timeout 300 python bench.py --config $c --wavelet cdf97 --no-cpu-baseline --no-e2e > gpurun_out/bench97_c$c.json 2> gpurun_out/bench97_c$c.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench97_c$c.json').read().strip().splitlines()[-1]); r=d['roofline']
print('9/7 c$c', round(d['value'],1), 'ms', round(d['ms_per_step'],4), 'k_ms', round(r['kernel_ms'],4), 'frac', round(r['frac'],3))" || tail -5 gpurun_out/bench97_c$c.err
done
for c in 1 2 3 4 5; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench_c$c.json').read().strip().splitlines()[-1]); r=d['roofline']
print('5/3 c$c', round(d['value'],1), 'ms', round(d['ms_per_step'],4), 'k_ms', round(r['kernel_ms'],4), 'frac', round(r['frac'],3))" || tail -5 gpurun_out/bench_c$c.err
done
