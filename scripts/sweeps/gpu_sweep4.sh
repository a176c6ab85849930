# c2 (4096^2, one level, cold) anomaly: tile heights, queue vs static, ring depth variants
mkdir -p gpurun_out
one() { timeout 200 python bench.py --config $1 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step']*1e3,1), round(d['roofline']['frac'],3))"; }
for tb in 3 7 11 15 23 31; do
  for mt in 1 100000; do
    echo "c2 MIN_TB=$tb MIN_TPW=$mt : $(DWT2_MIN_TB=$tb DWT2_MIN_TPW=$mt one 2)"
  done
done
for v in s3 s4 p2s4 w8; do
  for c in 2 3 4; do
    echo "variant $v c$c : $(DWT2_LIB=build/variants/libdwt2_$v.so one $c)"
  done
done
python scripts/level_times.py
