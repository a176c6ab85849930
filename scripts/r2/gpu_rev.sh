# Reverse tile order on every other pyramid level (DWT2_REV, tuning build):
# bench times of the multi-level configs, then per-launch DRAM bytes of one
# config-4 step with ncu's cache control OFF (the L2 hand-off between levels
# is the point; ncu's default flushes it between launches).  Never bench values.
V=build/variants/libdwt2_tuning.so
for r in 0 1 0 1; do out="rev $r:"; for c in 4 4b 5 2; do out="$out $(DWT2_REV=$r timeout 300 python bench.py --variant-lib $V --config $c --no-e2e --no-cpu-baseline --stat-steps 0 --no-gate | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('c$c', round(d['value'],1), round(d['ms_per_step']*1e3,1))")"; done; echo $out; done
mkdir -p gpurun_out/rev
for r in 0 1; do
DWT2_REV=$r timeout 600 ncu --clock-control none --cache-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -c 60 --csv \
  --log-file gpurun_out/rev/c4_rev$r.csv python bench.py --variant-lib $V --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-gate --stat-steps 0 --config 4 > /dev/null 2>&1; echo "ncu rev $r: $?"
done
