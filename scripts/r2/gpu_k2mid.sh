export DWT2_LIB=build/variants/libdwt2_tuning.so
SZ="4096 4096 8192 8192 2048 2048"
for mt in 16 12 8; do for tpw in 32 16; do echo "mintb $mt tpw $tpw: $(DWT2_K2_MINTB=$mt DWT2_K2_TPW=$tpw PROBE_WAVELET=cdf97 PROBE_COLD=1 timeout 200 python scripts/tile_probe.py $SZ)"; done; done
