export DWT2_LIB=build/variants/libdwt2_tuning.so
SZ="16384 16384 16384 8192 8192 8192"
for tb in 20 32 48 64; do echo "inv tb $tb: $(DWT2_K2INV_TB=$tb PROBE_OP=inverse PROBE_WAVELET=cdf97 timeout 200 python scripts/tile_probe.py $SZ)"; done
