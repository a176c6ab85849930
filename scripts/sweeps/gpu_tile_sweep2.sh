mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_inverse.py tests/test_gpu_schemes.py -q -x 2>&1 | tail -15
for combo in "32 11 2" "32 15 2" "32 23 2" "32 31 2" "24 15 2" "48 15 2"; do
  set -- $combo
  for c in 2 4 5 3; do
    r=$(DWT2_TPW=$1 DWT2_MIN_TB=$2 DWT2_MIN_TPW=$3 timeout 200 python bench.py --config $c --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step']*1e3,1), round(d['roofline']['frac'],3))")
    echo "TPW=$1 MINTB=$2 MINTPW=$3 config=$c : $r"
  done
done
