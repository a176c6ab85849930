timeout 300 python scripts/level_costs.py 8192 8192 8 cdf97 2>&1 | tail -8 | sed "s/.*: +//" | tr "\n" " "; echo
timeout 300 python scripts/level_costs.py 8192 8192 8 cdf97 inverse 2>&1 | tail -8 | sed "s/.*: +//" | tr "\n" " "; echo
export DWT2_LIB=build/variants/libdwt2_tuning.so
for q in 16384 262144; do echo "tail $q: $(DWT2_K2_TAIL_QUADS=$q timeout 300 python scripts/level_costs.py 8192 8192 8 cdf97 2>&1 | tail -8 | sed 's/.*: +//' | tr '\n' ' ')"; done
