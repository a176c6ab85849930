mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3
timeout 300 python __graft_entry__.py smoke | tail -1
for c in 5 3 4; do
  timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('c$c', round(d['value'],1), round(d['ms_per_step']*1e3,1), round(d['roofline']['frac'],3))"
done
ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -c 12 --csv --log-file gpurun_out/launches_c5_bulk.csv python bench.py --config 5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1
grep "gpu__time" gpurun_out/launches_c5_bulk.csv | head -8 | cut -c1-250
