for i in 1 2 3; do
for V in "" build/variants/libdwt2_p4s3.so build/variants/libdwt2_p4s4.so build/variants/libdwt2_p4s3w8.so; do
  VL=""; [ -n "$V" ] && VL="--variant-lib $V"
  echo "$V: $(timeout 300 python bench.py $VL --config 3 --no-e2e --no-cpu-baseline --no-gate --stat-steps 0 --steps 50 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step']*1e3,2), d['clocks']['sm_mhz'])") $(timeout 300 python bench.py $VL --config 5 --no-e2e --no-cpu-baseline --no-gate --stat-steps 0 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('c5', round(d['value'],1))")"
done; done
