# ncu evidence for profiles/round1: full captures of each kernel family, launch lists
mkdir -p gpurun_out/prof
P=gpurun_out/prof
N="ncu --clock-control none"
# 1. default bench command (config 3): launch list + one full capture of the level kernel
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > $P/plain_c3.json 2>&1 && \
$N --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -c 200 --csv --log-file $P/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1
$N --set full --import-source on -k regex:dwt53_level -s 3 -c 1 -o $P/full_c3_level python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > $P/full_c3.log 2>&1
# 2. config 4 (8 levels): per-level launch list
$N --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -c 200 --csv --log-file $P/launches_c4.csv python bench.py --config 4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1
# 3. config 5 (batched, 3 levels, odd 4095-wide images on the cp.async loader)
$N --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -c 200 --csv --log-file $P/launches_c5.csv python bench.py --config 5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > /dev/null 2>&1
# 4. CDF 9/7 level kernel, inverse ring kernel, scheme kernels (16384^2)
$N --set full --import-source on -k regex:dwt_k2 -s 1 -c 1 -o $P/full_c3_k2 python scripts/prof_target.py forward97 --reps 2 > $P/full_k2.log 2>&1
$N --set full --import-source on -k regex:inverse -s 1 -c 1 -o $P/full_c3_inverse python scripts/prof_target.py inverse --reps 2 > $P/full_inv.log 2>&1
for sch in sep_lifting sep_conv nonsep_lifting nonsep_adapted nonsep_naive; do
  $N --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file $P/launches_scheme_$sch.csv python scripts/prof_target.py scheme --scheme $sch --reps 1 > /dev/null 2>&1
done
ls -la $P
