P=gpurun_out/prof_r2b
mkdir -p $P
N="ncu --clock-control none"
timeout 900 $N --metrics gpu__time_duration.sum -c 400 --csv --log-file $P/launches_default_c3.csv \
  python bench.py --steps 2 --warmup 3 --stat-steps 0 --no-e2e --no-cpu-baseline > $P/launches_default_c3.log 2>&1; echo "default: $?"
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-gate --stat-steps 0"
timeout 900 $N --set full --import-source on -k regex:dwt53_level -s 3 -c 1 -o $P/c3 $B --config 3 > $P/c3.log 2>&1; echo "c3 full: $?"
timeout 900 $N --set full --import-source on -k regex:dwt_k2_level -s 3 -c 1 -o $P/c3_cdf97 $B --config 3 --wavelet cdf97 > $P/c397.log 2>&1; echo "c3 97 full: $?"
for c in 4 5; do
  timeout 900 $N --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -c 300 --csv \
    --log-file $P/launches_c$c.csv $B --config $c > /dev/null 2>&1; echo "launches c$c: $?"
done
timeout 900 $N --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -c 300 --csv \
    --log-file $P/launches_c4_cdf97.csv $B --config 4 --wavelet cdf97 > /dev/null 2>&1; echo "launches c4 97: $?"
timeout 900 python bench.py > $P/bench_default.json 2> $P/bench_default.err; tail -c 400 $P/bench_default.json
