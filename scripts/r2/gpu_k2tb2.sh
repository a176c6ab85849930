export DWT2_LIB=build/variants/libdwt2_tuning.so
for f in 1 2; do for q in 65536 262144; do echo "K2 smallf $f tail $q"; DWT2_K2_SMALLF=$f DWT2_K2_TAIL_QUADS=$q timeout 300 python scripts/level_costs.py 8192 8192 8 cdf97 2>&1 | tail -8 | awk '{print $NF, $0}' | cut -c1-90 | tr '\n' ' '; echo; done; done
