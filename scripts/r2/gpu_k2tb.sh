export DWT2_LIB=build/variants/libdwt2_tuning.so
for v in 0 1; do echo "K2 small tb $v"; DWT2_K2_SMALLTB=$v timeout 300 python scripts/level_costs.py 8192 8192 8 cdf97 2>&1 | tail -8; done
for v in 0 1; do echo "K2 small tb $v (4096^2 L1, 2048^2 L1)"; DWT2_K2_SMALLTB=$v PROBE_WAVELET=cdf97 PROBE_COLD=1 timeout 120 python scripts/tile_probe.py 4096 4096 2048 2048 16384 16384; done
