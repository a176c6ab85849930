# L2 policies of the level kernel (tuning build): DWT2_L2MODE bit 0 = input TMA
# loads evict_first, bit 1 = LL stores evict_last; DWT2_REV = reverse order on
# odd levels.  Bench times, then ncu DRAM bytes per launch with cache control off.
V=build/variants/libdwt2_tuning.so
for m in 0 1 2 3; do for r in 0 1; do out="l2mode $m rev $r:"; for c in 4 4b 5 3; do out="$out $(DWT2_REV=$r DWT2_L2MODE=$m timeout 300 python bench.py --variant-lib $V --config $c --no-e2e --no-cpu-baseline --stat-steps 0 --no-gate | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('c$c', round(d['value'],1), round(d['ms_per_step']*1e3,1))")"; done; echo $out; done; done
mkdir -p gpurun_out/l2mode
for m in 1 2 3; do
DWT2_REV=1 DWT2_L2MODE=$m timeout 600 ncu --clock-control none --cache-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -c 12 --csv \
  --log-file gpurun_out/l2mode/c4_m$m.csv python bench.py --variant-lib $V --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-gate --stat-steps 0 --config 4 > /dev/null 2>&1; echo "ncu m $m: $?"
done
