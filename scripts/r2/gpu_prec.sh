mkdir -p gpurun_out/r2i
for V in "" build/variants/libdwt2_f32.so; do
  if [ -n "$V" ]; then export DWT2_LIB=$V; TAG=fp32; VL="--variant-lib $V"; else unset DWT2_LIB; TAG=fp64; VL=""; fi
  for c in 3 2 4 4b; do timeout 300 python bench.py $VL --config $c --no-e2e --no-cpu-baseline --no-gate --stat-steps 0 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$TAG c$c 5/3', round(d['value'],1), round(d['ms_per_step']*1e3,2), round(d['roofline']['frac'],4))"; done
  for c in 3 4; do timeout 300 python bench.py $VL --config $c --wavelet cdf97 --no-e2e --no-cpu-baseline --no-gate --stat-steps 0 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$TAG c$c 9/7', round(d['value'],1), round(d['ms_per_step']*1e3,2), round(d['roofline']['frac'],4))"; done
  for c in 3 4; do timeout 300 python bench.py $VL --config $c --wavelet cdf97 --op inverse --no-e2e --no-cpu-baseline --no-gate --stat-steps 0 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$TAG c$c 9/7 inverse', round(d['value'],1), round(d['ms_per_step']*1e3,2), round(d['roofline']['frac'],4))"; done
  TAG=$TAG timeout 900 python scripts/r2/precision_probe.py
done
