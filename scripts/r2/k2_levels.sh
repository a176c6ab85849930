P=gpurun_out/r2j; mkdir -p $P
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv \
  --log-file $P/launches_c4_97.csv python bench.py --config 4 --wavelet cdf97 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-gate --stat-steps 0 > /dev/null 2>&1
echo rc $?
timeout 300 python scripts/level_costs.py 8192 8192 8 cdf97 2>&1 | tail -9; timeout 300 python scripts/level_costs.py 8192 8192 8 cdf53 2>&1 | tail -9
