set -x
python -c "from paper_1708_07853_b200 import _build; _build.build_variant('tuning', {'DWT2_TUNING': 1})"
timeout 900 python -m pytest tests/test_gpu_odd_pitch.py tests/test_gpu_parity.py tests/test_gpu_guard_bands.py -q -x 2>&1 | tail -2
for m in product off product off; do timeout 600 python scripts/r2/grp3_probe.py $m 2>&1 | tail -5; done
