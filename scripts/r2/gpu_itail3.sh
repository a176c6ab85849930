timeout 900 python -m pytest tests/test_gpu_inverse.py tests/test_gpu_wavelet97.py tests/test_gpu_fuzz.py -q -x 2>&1 | tail -2
export DWT2_LIB=build/variants/libdwt2_tuning.so
TAG=level DWT2_ITAIL_QUADS=0 DWT2_K2_ITAIL_QUADS=0 timeout 200 python scripts/r2/itail_probe.py
TAG=itail DWT2_ITAIL_QUADS=1000000 DWT2_K2_ITAIL_QUADS=1000000 timeout 200 python scripts/r2/itail_probe.py
for q in 0 16384 65536 262144; do echo "5/3 itail $q"; DWT2_ITAIL_QUADS=$q timeout 300 python scripts/level_costs.py 8192 8192 8 cdf53 inverse 2>&1 | tail -1; done
for q in 0 16384 65536 262144; do echo "9/7 itail $q"; DWT2_K2_ITAIL_QUADS=$q timeout 300 python scripts/level_costs.py 8192 8192 8 cdf97 inverse 2>&1 | tail -1; done
