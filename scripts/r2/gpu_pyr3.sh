set -x
mkdir -p gpurun_out/r2d
for V in tuning tuning_nopf; do
  export DWT2_LIB=build/variants/libdwt2_$V.so
  TAG=$V-base DWT2_PYRAMID=0 python scripts/r2/pyr_probe.py
  TAG=$V-pyr python scripts/r2/pyr_probe.py
  TAG=$V-pyr-uf0 DWT2_PYR_UNROLL_FIRST=0 python scripts/r2/pyr_probe.py
  TAG=$V-pyr-rmid8 DWT2_PYR_RMID=8 python scripts/r2/pyr_probe.py
  unset DWT2_LIB
  for c in 3 2; do python bench.py --variant-lib build/variants/libdwt2_$V.so --config $c --no-e2e --no-cpu-baseline --no-gate --stat-steps 0 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$V c$c', round(d['value'],1), round(d['ms_per_step']*1e3,2), round(d['roofline']['frac'],4))"; done
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:pyramid -s 3 -c 1 -o gpurun_out/r2d/pyr_c4 python bench.py --config 4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-gate --stat-steps 0 > gpurun_out/r2d/ncu_pyr.log 2>&1
