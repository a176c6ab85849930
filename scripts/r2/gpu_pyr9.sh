export DWT2_LIB=build/variants/libdwt2_prof.so
export DWT2_TAIL_QUADS=65536
export DWT2_PYRAMID=1
T="timeout 120"
TAG=pyr12 DWT2_PYR_MAXL=2 $T python scripts/r2/pyr_tiles.py 8192 8
TAG=pyr1 DWT2_PYR_MIN=1 DWT2_PYR_MAXL=1 $T python scripts/r2/pyr_tiles.py 8192 1
TAG=pyr2only DWT2_PYR_MIN=1 DWT2_PYR_MAXL=1 $T python scripts/r2/pyr_tiles.py 4096 1
