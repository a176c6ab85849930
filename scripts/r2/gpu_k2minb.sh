for V in "" build/variants/libdwt2_k2_minb5.so build/variants/libdwt2_k2_minb3.so; do
  VL=""; [ -n "$V" ] && VL="--variant-lib $V"
  for c in 3 4; do timeout 300 python bench.py $VL --config $c --wavelet cdf97 --no-e2e --no-cpu-baseline --no-gate --stat-steps 0 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$V c$c', round(d['value'],1), round(d['ms_per_step']*1e3,2), round(d['roofline']['frac'],4))"; done
  for c in 3 4; do timeout 300 python bench.py $VL --config $c --wavelet cdf97 --op inverse --no-e2e --no-cpu-baseline --no-gate --stat-steps 0 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$V inv c$c', round(d['value'],1), round(d['ms_per_step']*1e3,2), round(d['roofline']['frac'],4))"; done
done
