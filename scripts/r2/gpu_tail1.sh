mkdir -p gpurun_out/r2f
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_odd_pitch.py tests/test_gpu_guard_bands.py -q -x 2>&1 | tail -4
export DWT2_LIB=build/variants/libdwt2_tuning.so
TAG=notail DWT2_TAIL_QUADS=0 python scripts/r2/pyr_probe.py
TAG=tail python scripts/r2/pyr_probe.py
TAG=tail-16k DWT2_TAIL_QUADS=16384 python scripts/r2/pyr_probe.py
TAG=tail-64k DWT2_TAIL_QUADS=65536 python scripts/r2/pyr_probe.py
TAG=tail-1m DWT2_TAIL_QUADS=1048576 python scripts/r2/pyr_probe.py
TAG=tail-cta1 DWT2_TAIL_CTAS=1 python scripts/r2/pyr_probe.py
TAG=tail-cta4 DWT2_TAIL_CTAS=4 python scripts/r2/pyr_probe.py
TAG=notail DWT2_TAIL_QUADS=0 python scripts/launch_floor.py
TAG=tail python scripts/launch_floor.py
unset DWT2_LIB
for c in 4 4b 1; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/r2f/fwd53_c$c.json 2>gpurun_out/r2f/fwd53_c$c.err; python -c "import json; d=json.loads(open('gpurun_out/r2f/fwd53_c$c.json').read().strip().splitlines()[-1]); print('c$c', round(d['value'],1), round(d['ms_per_step']*1e3,2), d['gate']['status'], d['step_stats'].get('median_ms'))"; done
