export DWT2_LIB=build/variants/libdwt2_tuning.so
TAG=level DWT2_ITAIL_QUADS=0 DWT2_K2_ITAIL_QUADS=0 timeout 200 python scripts/r2/itail_probe.py
TAG=itail DWT2_ITAIL_QUADS=1000000 DWT2_K2_ITAIL_QUADS=1000000 timeout 200 python scripts/r2/itail_probe.py
timeout 300 ncu --set full -k regex:itail -c 1 -o gpurun_out/r2k_itail python scripts/r2/itail_probe.py > /dev/null 2>&1
