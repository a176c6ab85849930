timeout 900 python -m pytest tests/test_gpu_inverse.py tests/test_gpu_odd_pitch.py tests/test_gpu_guard_bands.py tests/test_gpu_fuzz.py -q -x 2>&1 | tail -3
TAG=bulk timeout 200 python scripts/r2/inv_probe.py
DWT2_LIB=build/variants/libdwt2_tuning.so DWT2_INV_BULK=0 TAG=ldg timeout 200 python scripts/r2/inv_probe.py
for v in ib_minb4 ib_bds6 ib_bds3; do DWT2_LIB=build/variants/libdwt2_$v.so TAG=$v timeout 200 python scripts/r2/inv_probe.py; done
