TAG=prod timeout 200 python scripts/r2/inv_probe.py
for v in inv_pf1_b1 inv_pf2_b1 inv_pf3_b1; do DWT2_LIB=build/variants/libdwt2_$v.so TAG=$v timeout 200 python scripts/r2/inv_probe.py; done
