mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_wavelet97.py tests/test_gpu_inverse.py -q -x 2>&1 | tail -3
for c in 3 4; do
  timeout 300 python bench.py --config $c --wavelet cdf97 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('9/7 c$c', round(d['value'],1), round(d['ms_per_step']*1e3,1), round(d['roofline']['frac'],3))"
done
timeout 600 python scripts/inverse_bench.py > gpurun_out/inverse_bench.log 2>&1; python -c "
import json
for l in open('gpurun_out/inverse_bench.log'):
    d=json.loads(l); print('inv', d['config'], round(d['inverse_us'],1), 'us, level1 frac', round(d['inverse_level1_frac_of_copy'],3), 'fwd', round(d['forward_us'],1))"
