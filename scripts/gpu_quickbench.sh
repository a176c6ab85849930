set -x
for i in 1 2; do timeout 120 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('DEFAULT', d['value'], d['roofline']['frac'])"; done
for v in build/variants/*.so; do
  for i in 1 2; do DWT2_LIB=$v timeout 120 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['roofline']['frac'])"; done
done
