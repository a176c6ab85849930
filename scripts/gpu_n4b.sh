mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_wavelet97.py -q -x 2>&1 | tail -15
for c in 1 2 3 4 5; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench_c$c.json').read().strip().splitlines()[-1]); r=d['roofline']
print('5/3 c$c', round(d['value'],1), 'ms', round(d['ms_per_step'],4), 'k_ms', round(r['kernel_ms'],4), 'frac', round(r['frac'],3))" || tail -5 gpurun_out/bench_c$c.err
done
timeout 300 python bench.py --config 2 --wavelet cdf97 --no-cpu-baseline --no-e2e | tail -1 | cut -c1-300
ncu --set full --clock-control none --import-source on -k regex:dwt_k2 -s 3 -c 1 -o gpurun_out/prof_k2_c3 python bench.py --config 3 --wavelet cdf97 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/ncu_k2.log 2>&1; tail -3 gpurun_out/ncu_k2.log
ncu --set full --clock-control none --import-source on -k regex:inverse -s 3 -c 1 -o gpurun_out/prof_inv_c3 python scripts/inverse_bench.py --iters 2 > gpurun_out/ncu_inv.log 2>&1; tail -3 gpurun_out/ncu_inv.log
