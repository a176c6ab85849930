export DWT2_LIB=build/variants/libdwt2_tuning.so
python -c "
import torch; p=torch.cuda.get_device_properties(0); print(p.name, 'L2', p.L2_cache_size)
from cuda.bindings import runtime as rt
print('max persisting', rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxPersistingL2CacheSize, 0), 'max window', rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxAccessPolicyWindowSize, 0))
" 2>&1 | tail -2
TAG=base timeout 120 python scripts/r2/pyr_probe.py
for mb in 32 64 96; do TAG=persist$mb DWT2_L2_PERSIST=1 DWT2_L2_SETASIDE_MB=$mb timeout 120 python scripts/r2/pyr_probe.py; done
TAG=setaside-only DWT2_L2_SETASIDE_MB=64 timeout 120 python scripts/r2/pyr_probe.py
