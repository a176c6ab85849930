# re-capture of the 5/3 level kernel workloads after the tile-decode changes
# (fast division, unrolled first stage on guided / static / row-grouped launches)
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
cap c1 dwt53_level 3 --config 1
cap c2 dwt53_level 3 --config 2
cap c3 dwt53_level 3 --config 3
cap c4 dwt53_level 24 --config 4
cap c4b dwt53_level 24 --config 4b
cap c5 dwt53_level 18 --config 5
cap c5_group2 dwt53_level 21 --config 5
