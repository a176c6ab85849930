mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wavelet97.py -q -x 2>&1 | tail -2
for v in k2q2 k2q4b3 k2q4b2; do
  for c in 3 4; do
    echo "$v c$c: $(timeout 300 python bench.py --variant-lib build/variants/libdwt2_$v.so --config $c --wavelet cdf97 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step']*1e3,1), round(d['roofline']['frac'],3))")"
  done
done
