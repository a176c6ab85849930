export DWT2_LIB=build/variants/libdwt2_tuning.so
SZ="16384 16384 8192 8192 4096 4096"
for cfg in "32 16" "16 16" "8 16" "16 24" "8 32" "32 12"; do set -- $cfg
  echo "fwd tpw $1 mintb $2: $(DWT2_K2_TPW=$1 DWT2_K2_MINTB=$2 PROBE_WAVELET=cdf97 PROBE_COLD=1 timeout 200 python scripts/tile_probe.py $SZ)"
done
for cfg in "8 16 20" "16 16 20" "8 16 32" "8 16 12" "4 16 0"; do set -- $cfg
  echo "inv tpw $1 mintb $2 tb $3: $(DWT2_K2INV_TPW=$1 DWT2_K2INV_MINTB=$2 DWT2_K2INV_TB=$3 PROBE_OP=inverse PROBE_WAVELET=cdf97 timeout 200 python scripts/tile_probe.py $SZ)"
done
