set -x
for v in build/variants/*.so; do
  echo "== $v"
  DWT2_LIB=$v timeout 120 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('RESULT', d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
./scripts/membench > gpurun_out/membench.txt 2>&1 && \
timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.per_cycle_active --csv --log-file gpurun_out/membench_ncu.csv ./scripts/membench > /dev/null 2>&1
for v in build/variants/libdwt2_nm32_p8s2.so build/variants/libdwt2_fp64_p4s4m3.so; do
DWT2_LIB=$v timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.per_cycle_active -k regex:dwt53 -s 2 -c 1 --csv --log-file gpurun_out/ncu_$(basename $v).csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
ls gpurun_out
