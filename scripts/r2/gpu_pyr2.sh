set -x
mkdir -p gpurun_out/r2c
V=build/variants/libdwt2_tuning.so
export DWT2_LIB=$V
TAG=base DWT2_PYRAMID=0 python scripts/r2/pyr_probe.py
TAG=pyr python scripts/r2/pyr_probe.py
TAG=pyr_big DWT2_PYR_RMID=1 DWT2_PYR_RSMALL=1 python scripts/r2/pyr_probe.py
TAG=pyr_small7 DWT2_PYR_RMID=100000 DWT2_PYR_RSMALL=1 python scripts/r2/pyr_probe.py
TAG=pyr_uf0 DWT2_PYR_UNROLL_FIRST=0 python scripts/r2/pyr_probe.py
unset DWT2_LIB
python bench.py --config 4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-gate --stat-steps 0 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:pyramid -s 3 -c 1 -o gpurun_out/r2c/pyr_c4 python bench.py --config 4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-gate --stat-steps 0 > gpurun_out/r2c/ncu_pyr.log 2>&1
DWT2_LIB=$V DWT2_PYRAMID=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:level_kernel -s 24 -c 2 -o gpurun_out/r2c/lvl_c4 python bench.py --variant-lib $V --config 4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-gate --stat-steps 0 > gpurun_out/r2c/ncu_lvl.log 2>&1
ls -la gpurun_out/r2c
