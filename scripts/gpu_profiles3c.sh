# re-capture of the kernels whose tile policy changed after gpu_profiles3.sh
# (15-row tiles on large 5/3 levels: config 5; inverse 20-row tiles; K = 2
# tiles): same commands, same names
P=gpurun_out/prof3
mkdir -p $P
N="ncu --clock-control none"
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph"
cap() {
  name=$1; kern=$2; skip=$3; shift 3
  rm -f $P/$name.ncu-rep
  timeout 900 $N --set full --import-source on -k regex:$kern -s $skip -c 1 -o $P/$name $B "$@" > $P/$name.log 2>&1
  echo "$name: rc=$?"
}
cap c5 dwt53_level 18 --config 5
cap c5_group2 dwt53_level 21 --config 5
cap c3_inverse inverse 3 --config 3 --op inverse
cap c4_inverse inverse 31 --config 4 --op inverse
cap c3_cdf97 dwt_k2_level 3 --config 3 --wavelet cdf97
cap c3_cdf97_inverse dwt_k2_inverse 3 --config 3 --wavelet cdf97 --op inverse
timeout 600 $N --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -c 200 --csv \
  --log-file $P/launches_c5.csv $B --config 5 > /dev/null 2>&1
