timeout 900 python -m pytest tests/test_gpu_wavelet97.py tests/test_gpu_fuzz.py tests/test_gpu_guard_bands.py -q -x 2>&1 | tail -1
export DWT2_LIB=build/variants/libdwt2_tuning.so
SZ="4096 4096 8192 8192 2048 2048 16384 16384"
for ef in 0 1; do echo "inv edgefirst $ef: $(DWT2_K2INV_EDGEFIRST=$ef PROBE_OP=inverse PROBE_WAVELET=cdf97 timeout 200 python scripts/tile_probe.py $SZ)"; done
unset DWT2_LIB
for c in 3 4; do timeout 300 python bench.py --config $c --wavelet cdf97 --op inverse --no-e2e --no-cpu-baseline --stat-steps 0 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('inv c$c', round(d['value'],1), round(d['ms_per_step']*1e3,2), d['gate']['status'])"; done
