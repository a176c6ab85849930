set -x
export DWT2_LIB=build/variants/libdwt2_prof.so
TAG=prof python scripts/r2/pyr_levels.py 8192 8
TAG=prof python scripts/r2/pyr_levels.py 2048 3 64
TAG=prof-rmid8 DWT2_PYR_RMID=8 python scripts/r2/pyr_levels.py 8192 8
export DWT2_LIB=build/variants/libdwt2_tuning.so
TAG=base DWT2_PYRAMID=0 python scripts/r2/pyr_probe.py
TAG=pyr python scripts/r2/pyr_probe.py
