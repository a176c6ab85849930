# second pass of gpu_profiles3.sh: config 5's second group (32 x 4095x3001,
# level 1 = launch 4 of each step) and config 4's level-1 inverse (the last of
# the 8 launches of each inverse step)
P=gpurun_out/prof3
mkdir -p $P
N="ncu --clock-control none"
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph"
timeout 900 $N --set full --import-source on -k regex:dwt53_level -s 21 -c 1 -o $P/c5_group2 $B --config 5 > $P/c5_group2.log 2>&1; echo "c5_group2 rc=$?"
timeout 900 $N --set full --import-source on -k regex:inverse -s 31 -c 1 -o $P/c4_inverse $B --config 4 --op inverse > $P/c4_inverse.log 2>&1; echo "c4_inverse rc=$?"
