export DWT2_LIB=build/variants/libdwt2_tuning.so
for f in 0 1; do for q in 0 65536; do echo "K2INV smallf $f itail $q"; DWT2_K2INV_SMALLF=$f DWT2_K2_ITAIL_QUADS=$q timeout 300 python scripts/level_costs.py 8192 8192 8 cdf97 inverse 2>&1 | tail -8 | sed 's/.*: +//' | tr '\n' ' '; echo; done; done
