timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for ef in 0 1; do out="ef $ef:"; for c in 3 2 4 4b 5; do out="$out $(DWT2_EDGEFIRST=$ef timeout 300 python bench.py --variant-lib build/variants/libdwt2_tuning.so --config $c --no-e2e --no-cpu-baseline --stat-steps 0 --no-gate | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('c$c', round(d['value'],1))")"; done; echo $out; done
for ef in 0 1; do echo "ef $ef inv: $(DWT2_EDGEFIRST=$ef PROBE_OP=inverse timeout 200 python scripts/tile_probe.py 4096 4096 8192 8192)"; done
