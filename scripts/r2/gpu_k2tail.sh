timeout 900 python -m pytest tests/test_gpu_wavelet97.py tests/test_gpu_fuzz.py tests/test_gpu_tail.py tests/test_gpu_guard_bands.py -q -x 2>&1 | tail -3
export DWT2_LIB=build/variants/libdwt2_tuning.so
for q in 0 16384 65536 262144 1048576; do echo "K2 tail quads $q"; DWT2_K2_TAIL_QUADS=$q timeout 300 python scripts/level_costs.py 8192 8192 8 cdf97 2>&1 | tail -1; done
unset DWT2_LIB
timeout 300 python bench.py --config 4 --wavelet cdf97 --no-cpu-baseline | tail -c 600
