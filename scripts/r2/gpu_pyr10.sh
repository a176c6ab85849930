mkdir -p gpurun_out/r2g
export DWT2_LIB=build/variants/libdwt2_prof.so
export DWT2_TAIL_QUADS=65536
export DWT2_PYRAMID=1
T="timeout 120"
TAG=pyr12 OUT=gpurun_out/r2g/pyr12.npz DWT2_PYR_MAXL=2 $T python scripts/r2/pyr_tiles.py 8192 8
TAG=pyrall OUT=gpurun_out/r2g/pyrall.npz $T python scripts/r2/pyr_tiles.py 8192 8
