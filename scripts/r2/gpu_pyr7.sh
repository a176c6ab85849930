mkdir -p gpurun_out/r2e
export DWT2_LIB=build/variants/libdwt2_tuning.so
timeout 600 ncu --set full --import-source on --clock-control none -k regex:pyramid -s 2 -c 1 -o gpurun_out/r2e/pyr_c5g python scripts/r2/pyr_once.py 2048 3 64 > gpurun_out/r2e/ncu1.log 2>&1
DWT2_PYRAMID=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:level_kernel -s 6 -c 3 -o gpurun_out/r2e/lvl_c5g python scripts/r2/pyr_once.py 2048 3 64 > gpurun_out/r2e/ncu2.log 2>&1
ls -la gpurun_out/r2e
