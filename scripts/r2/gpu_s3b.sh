timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for c in 3 5 2 4; do timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline --stat-steps 0 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('c$c', round(d['value'],1), round(d['ms_per_step']*1e3,2), round(d['roofline']['frac'],4), d['gate']['status'])"; done
PROBE_COLD=1 timeout 200 python scripts/tile_probe.py 16384 16384 16384 8192 16384 2048 20000 8000
