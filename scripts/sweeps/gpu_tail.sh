# small tiles at the end of the queue on large levels (DWT2_TAIL percent)
b() { timeout 300 python bench.py "$@" --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1), round(d['roofline']['frac'],4))"; }
for t in 0 3 6 10 15; do echo "TAIL=$t c3: $(DWT2_TAIL=$t b --config 3 --steps 40)  c4: $(DWT2_TAIL=$t b --config 4)  c5: $(DWT2_TAIL=$t b --config 5)"; done
for t in 0 3 6 10 15; do echo "TAIL=$t c3 again: $(DWT2_TAIL=$t b --config 3 --steps 40)"; done
