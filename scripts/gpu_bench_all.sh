set -x
timeout 600 python -m pytest tests -m gpu -q -x -k "tiny or config1 or config4 or config5 or host or strips_equal" 2>&1 | tail -3; [ ${PIPESTATUS[0]} -eq 0 ] || exit 1
for c in 3 1 2 4 4b 5; do timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('CONFIG', d['config']['workload'][:32], round(d['value'],1), 'ms', round(d['ms_per_step'],4), 'l1frac', round(d['roofline']['frac'],3), 'l1ms', round(d['roofline']['kernel_ms'],4), d.get('launch'))"; done
timeout 300 python bench.py --config 4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/plain4.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:dwt53 --csv --log-file gpurun_out/launches_c4.csv python bench.py --config 4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1
ls gpurun_out
