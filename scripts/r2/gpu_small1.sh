export DWT2_LIB=build/variants/libdwt2_tuning.so
export DWT2_TAIL_QUADS=65536
T="timeout 200"
SZ="16384 16384 8192 8192 16384 8192 16384 2048 4096 4096"
for cfg in "0 3" "1 3" "2 3" "4 3" "1 7" "2 7" "3 7"; do set -- $cfg
  TAG="small tpw$1 tb$2" DWT2_SMALL_TPW=$1 DWT2_SMALL_TB=$2 PROBE_COLD=1 $T python scripts/tile_probe.py $SZ
  TAG="small tpw$1 tb$2" DWT2_SMALL_TPW=$1 DWT2_SMALL_TB=$2 $T python scripts/r2/pyr_probe.py
done
