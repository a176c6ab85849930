timeout 900 python -m pytest tests/test_gpu_inverse.py tests/test_gpu_wavelet97.py tests/test_gpu_fuzz.py tests/test_gpu_odd_pitch.py -q -x 2>&1 | tail -1
export DWT2_LIB=build/variants/libdwt2_tuning.so
for v in 0 1; do for q in 0 16384; do echo "5/3 inv small $v itail $q"; DWT2_INV_SMALL=$v DWT2_ITAIL_QUADS=$q timeout 300 python scripts/level_costs.py 8192 8192 8 cdf53 inverse 2>&1 | tail -8 | sed 's/.*: +//' | tr '\n' ' '; echo; done; done
echo "9/7 inverse (product)"; unset DWT2_LIB; timeout 300 python scripts/level_costs.py 8192 8192 8 cdf97 inverse 2>&1 | tail -1
