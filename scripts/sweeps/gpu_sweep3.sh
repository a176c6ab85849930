mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wavelet97.py -q -x 2>&1 | tail -2
for c in 3 4; do
  timeout 300 python bench.py --config $c --wavelet cdf97 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('9/7 c$c', round(d['value'],1), round(d['ms_per_step']*1e3,1), round(d['roofline']['frac'],3))"
done
for mt in 2 4 6 8 12; do
  for c in 2 4 5 3; do
    r=$(DWT2_MIN_TPW=$mt timeout 200 python bench.py --config $c --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step']*1e3,1), round(d['roofline']['frac'],3))")
    echo "MIN_TPW=$mt config=$c : $r"
  done
done
