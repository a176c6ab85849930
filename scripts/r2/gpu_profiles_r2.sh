# Round 2 ncu evidence of the current build (profiles/round2): launch lists of the
# default bench command and of configs 4 / 4b / 5 (the contract's
# gpu__time_duration pass), one --set full capture of the config-3 level kernel
# and of the config-4 tail kernel.  Never a bench value.
P=gpurun_out/prof_r2
mkdir -p $P
N="ncu --clock-control none"
timeout 900 $N --metrics gpu__time_duration.sum -c 400 --csv --log-file $P/launches_default_c3.csv \
  python bench.py --steps 2 --warmup 3 --stat-steps 0 --no-e2e --no-cpu-baseline > $P/launches_default_c3.log 2>&1; echo "default: $?"
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph --no-gate --stat-steps 0"
for c in 4 4b 5; do
  timeout 900 $N --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -c 300 --csv \
    --log-file $P/launches_c$c.csv $B --config $c > /dev/null 2>&1; echo "launches c$c: $?"
done
timeout 900 $N --set full --import-source on -k regex:dwt53_level -s 3 -c 1 -o $P/c3 $B --config 3 > $P/c3.log 2>&1; echo "c3 full: $?"
timeout 900 $N --set full --import-source on -k regex:tail -s 3 -c 1 -o $P/c4_tail $B --config 4 > $P/c4_tail.log 2>&1; echo "c4 tail full: $?"
ls -la $P
