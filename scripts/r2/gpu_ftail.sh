timeout 900 python -m pytest tests/test_gpu_tail.py tests/test_gpu_wavelet97.py -q -x 2>&1 | tail -2
export DWT2_LIB=build/variants/libdwt2_tuning.so
for q in 65536 262144; do echo "9/7 fwd tail $q"; DWT2_K2_TAIL_QUADS=$q timeout 300 python scripts/level_costs.py 8192 8192 8 cdf97 2>&1 | tail -1; done
for q in 0 16384 65536; do echo "5/3 fwd tail $q"; DWT2_TAIL_QUADS=$q timeout 300 python scripts/level_costs.py 8192 8192 8 cdf53 2>&1 | tail -1; done
DWT2_TAIL_QUADS=0 TAG=notail timeout 120 python scripts/launch_floor.py 2>&1 | head -3
DWT2_TAIL_QUADS=1000000 TAG=tail timeout 120 python scripts/launch_floor.py 2>&1 | head -5
