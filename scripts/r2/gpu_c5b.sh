set -x
for v in product build/variants/libdwt2_old.so build/variants/libdwt2_nohooks.so product build/variants/libdwt2_old.so build/variants/libdwt2_nohooks.so; do timeout 600 python scripts/r2/c5_groups.py $v 2>&1 | tail -4; done
