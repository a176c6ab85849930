timeout 900 python -m pytest tests/test_gpu_inverse.py tests/test_gpu_guard_bands.py -q -x 2>&1 | tail -2
timeout 600 python scripts/inverse_bench.py > gpurun_out/inverse_bench.log 2>&1; python -c "
import json
for l in open('gpurun_out/inverse_bench.log'):
    d=json.loads(l); print('inv', d['config'], round(d['inverse_us'],1), 'us, level1 frac', round(d['inverse_level1_frac_of_copy'],3), 'fwd', round(d['forward_us'],1))"
