export DWT2_LIB=build/variants/libdwt2_tuning.so
export DWT2_TAIL_QUADS=65536
T="timeout 120"
TAG=base $T python scripts/r2/pyr_probe.py
TAG=pyr12 DWT2_PYRAMID=1 DWT2_PYR_MAXL=2 $T python scripts/r2/pyr_probe.py
TAG=pyr123 DWT2_PYRAMID=1 DWT2_PYR_MAXL=3 $T python scripts/r2/pyr_probe.py
TAG=pyr1234 DWT2_PYRAMID=1 DWT2_PYR_MAXL=4 $T python scripts/r2/pyr_probe.py
TAG=pyr234 DWT2_PYRAMID=1 DWT2_PYR_FIRST=1 DWT2_PYR_MAXL=3 $T python scripts/r2/pyr_probe.py
TAG=pyr23 DWT2_PYRAMID=1 DWT2_PYR_FIRST=1 DWT2_PYR_MAXL=2 $T python scripts/r2/pyr_probe.py
TAG=pyr34 DWT2_PYRAMID=1 DWT2_PYR_FIRST=2 DWT2_PYR_MAXL=2 $T python scripts/r2/pyr_probe.py
TAG=pyrall DWT2_PYRAMID=1 $T python scripts/r2/pyr_probe.py
TAG=tail-cta1 DWT2_TAIL_CTAS=1 $T python scripts/r2/pyr_probe.py
TAG=tail-cta3 DWT2_TAIL_CTAS=3 $T python scripts/r2/pyr_probe.py
TAG=notail DWT2_TAIL_QUADS=0 $T python scripts/launch_floor.py
TAG=tail DWT2_TAIL_QUADS=262144 $T python scripts/launch_floor.py
