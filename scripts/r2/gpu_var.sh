set -x
for v in product build/variants/libdwt2_pairs2.so build/variants/libdwt2_minb5.so product; do timeout 600 python scripts/r2/variant_probe.py $v 2>&1 | tail -5; done
