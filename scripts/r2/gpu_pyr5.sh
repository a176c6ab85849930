export DWT2_LIB=build/variants/libdwt2_tuning.so
TAG=level python scripts/r2/pyr_single.py
TAG=pyr1 DWT2_PYR_MIN=1 python scripts/r2/pyr_single.py
TAG=pyr1-pub DWT2_PYR_MIN=1 DWT2_PYR_PUBLAST=1 python scripts/r2/pyr_single.py
TAG=base DWT2_PYRAMID=0 python scripts/r2/pyr_probe.py
TAG=pyr python scripts/r2/pyr_probe.py
TAG=pyr-pubeach DWT2_PYR_PUBEACH=1 python scripts/r2/pyr_probe.py
export DWT2_LIB=build/variants/libdwt2_prof.so
TAG=prof python scripts/r2/pyr_levels.py 8192 8
TAG=prof python scripts/r2/pyr_levels.py 2048 3 64
