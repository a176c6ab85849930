export DWT2_LIB=build/variants/libdwt2_tuning.so
TAG=base DWT2_PYRAMID=0 python scripts/r2/pyr_probe.py
TAG=pyr python scripts/r2/pyr_probe.py
TAG=pyr-tpw2 DWT2_PYR_TPW=2 python scripts/r2/pyr_probe.py
TAG=pyr-tpw8 DWT2_PYR_TPW=8 python scripts/r2/pyr_probe.py
TAG=pyr-large4 DWT2_PYR_LARGE=4 python scripts/r2/pyr_probe.py
TAG=pyr-large16 DWT2_PYR_LARGE=16 python scripts/r2/pyr_probe.py
TAG=pyr1 DWT2_PYR_MIN=1 python scripts/r2/pyr_single.py
export DWT2_LIB=build/variants/libdwt2_prof.so
TAG=prof python scripts/r2/pyr_levels.py 8192 8
TAG=prof python scripts/r2/pyr_levels.py 2048 3 64
