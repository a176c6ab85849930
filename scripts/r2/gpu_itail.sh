timeout 900 python -m pytest tests/test_gpu_inverse.py tests/test_gpu_wavelet97.py tests/test_gpu_fuzz.py tests/test_gpu_odd_pitch.py tests/test_gpu_guard_bands.py -q -x 2>&1 | tail -3
export DWT2_LIB=build/variants/libdwt2_tuning.so
for q in 0 16384 65536 262144; do echo "5/3 itail $q"; DWT2_ITAIL_QUADS=$q timeout 300 python scripts/level_costs.py 8192 8192 8 cdf53 inverse 2>&1 | tail -1; done
for q in 0 65536 262144 1048576; do echo "9/7 itail $q"; DWT2_K2_ITAIL_QUADS=$q timeout 300 python scripts/level_costs.py 8192 8192 8 cdf97 inverse 2>&1 | tail -1; done
