set -x
python -c "from paper_1708_07853_b200 import _build; _build.build_variant('tuning', {'DWT2_TUNING': 1})"
timeout 900 python -m pytest tests/test_gpu_inverse.py tests/test_gpu_wavelet97.py tests/test_gpu_odd_pitch.py tests/test_gpu_fuzz.py -q -x 2>&1 | tail -3
for m in 0 65536 262144 1048576; do timeout 600 python scripts/r2/inv_small_probe.py $m 2>&1 | tail -5; done
