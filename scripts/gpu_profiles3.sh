# ncu evidence of the current build (profiles/round1/session3): one --set full
# capture of the level-1 (dominant) kernel of every bench workload, in the
# launch configuration bench.py times (--no-graph: the same launches, issued
# one by one so ncu can replay them), and per-launch lists of the multi-level
# configs.  Never a bench value: ncu serialises and flushes caches.
P=gpurun_out/prof3
mkdir -p $P
N="ncu --clock-control none"
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph"
cap() {   # name kernel-regex launches-to-skip bench-args...
  name=$1; kern=$2; skip=$3; shift 3
  timeout 900 $N --set full --import-source on -k regex:$kern -s $skip -c 1 -o $P/$name $B "$@" > $P/$name.log 2>&1
  echo "$name: rc=$?"
}
cap c1 dwt53_level 3 --config 1
cap c2 dwt53_level 3 --config 2
cap c3 dwt53_level 3 --config 3
cap c4 dwt53_level 24 --config 4
cap c4b dwt53_level 24 --config 4b
cap c5 dwt53_level 18 --config 5
cap c3_inverse inverse 3 --config 3 --op inverse
cap c4_inverse inverse 24 --config 4 --op inverse
cap c3_cdf97 dwt_k2_level 3 --config 3 --wavelet cdf97
cap c3_cdf97_inverse dwt_k2_inverse 3 --config 3 --wavelet cdf97 --op inverse
for c in 4 4b 5; do
  timeout 600 $N --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -c 200 --csv \
    --log-file $P/launches_c$c.csv $B --config $c > /dev/null 2>&1
done
ls -la $P
