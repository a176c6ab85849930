set -x
timeout 300 python __graft_entry__.py smoke
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 900 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('default', d['value'], d['ms_per_step'], d['roofline']['frac'], d['gate']['status'], d['e2e']['value'], d['clocks'])"
