mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_strip_levels.py -q -x 2>&1 | tail -15
for c in 1 2 3 4; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench_c$c.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$c', round(d['value'],1), 'ms', round(d['ms_per_step'],4), 'k_ms', round(r['kernel_ms'],4), 'frac', round(r['frac'],3), d['config']['l2'])"
done
timeout 900 python scripts/scheme_compare.py --iters 20 > gpurun_out/scheme_compare.log 2>&1; tail -8 gpurun_out/scheme_compare.log
timeout 600 python scripts/inverse_bench.py > gpurun_out/inverse_bench.log 2>&1; cut -c1-250 gpurun_out/inverse_bench.log
