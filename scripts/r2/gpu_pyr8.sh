export DWT2_TAIL_QUADS=65536
T="timeout 120"
for V in tuning t_r2 t_r0 t_r0w0; do
export DWT2_LIB=build/variants/libdwt2_$V.so
TAG=$V-base $T python scripts/r2/pyr_probe.py
TAG=$V-pyr12 DWT2_PYRAMID=1 DWT2_PYR_MAXL=2 $T python scripts/r2/pyr_probe.py
TAG=$V-pyrall DWT2_PYRAMID=1 $T python scripts/r2/pyr_probe.py
done
