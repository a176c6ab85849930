set -x
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4; [ ${PIPESTATUS[0]} -eq 0 ] || exit 1
timeout 120 python bench.py --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | tail -1
for v in build/variants/*.so; do
  echo "== $v"
  DWT2_LIB=$v timeout 120 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('RESULT', d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
for c in 1 2 4 5; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('CONFIG', d['config']['workload'][:30], d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'])"; done
