set -x
python -c "from paper_1708_07853_b200 import _build; _build.build_variant('tuning', {'DWT2_TUNING': 1})"
timeout 900 python -m pytest tests/test_gpu_wavelet97.py tests/test_gpu_tail.py -q -x 2>&1 | tail -2
for m in 0 262144 1048576 4194304; do DWT2_K2_TAIL_QUADS=4096 timeout 600 python scripts/r2/k2small_probe.py $m 2>&1 | tail -5; done
