export DWT2_LIB=build/variants/libdwt2_tuning.sh
export DWT2_LIB=build/variants/libdwt2_tuning.so
SZ="8192 8192 8192 4096 16384 2048"
for g in 8 12 16; do for a in 60 80; do echo "maxtpw $g guided_a $a: $(DWT2_GUIDED_MAXTPW=$g DWT2_GUIDED_A=$a PROBE_COLD=1 timeout 200 python scripts/tile_probe.py $SZ)"; done; done
