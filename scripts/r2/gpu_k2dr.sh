for V in "" k2dr2 k2dr3; do
  VL=""; [ -n "$V" ] && VL="--variant-lib build/variants/libdwt2_$V.so"
  out="$V:"; for op in forward inverse; do for c in 3 4; do out="$out $(timeout 300 python bench.py $VL --config $c --wavelet cdf97 --op $op --no-e2e --no-cpu-baseline --stat-steps 0 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$op c$c', round(d['value'],1), d['gate']['status'])")"; done; done; echo $out
done
