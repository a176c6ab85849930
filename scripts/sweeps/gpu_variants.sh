set -x
timeout 900 python -m pytest tests -m gpu -q -x -k "tiny or ragged or config1 or config4 or strips_equal or config5" 2>&1 | tail -3; [ ${PIPESTATUS[0]} -eq 0 ] || exit 1
for v in build/variants/*.so; do
  echo "== $v"
  case $v in *prof*) DWT2_LIB=$v timeout 120 python scripts/prof_waits.py; continue;; esac
  DWT2_LIB=$v timeout 60 python __graft_entry__.py smoke 2>&1 | tail -1
  timeout 120 python bench.py --variant-lib $v --steps 50 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('RESULT', d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
