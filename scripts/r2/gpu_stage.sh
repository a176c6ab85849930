for V in "" build/variants/libdwt2_p2s2.so build/variants/libdwt2_p2s3.so build/variants/libdwt2_p2s4.so build/variants/libdwt2_p4s3.so; do
  VL=""; [ -n "$V" ] && VL="--variant-lib $V"
  out="$V:"
  for c in 3 2 4 1; do out="$out $(timeout 300 python bench.py $VL --config $c --no-e2e --no-cpu-baseline --stat-steps 0 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('c$c', round(d['value'],1), round(d['ms_per_step']*1e3,2), d['gate']['status'])")"; done
  echo $out
done
