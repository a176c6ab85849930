set -x
python -c "from paper_1708_07853_b200 import _build; _build.build_variant('tuning', {'DWT2_TUNING': 1})"
for m in product 1073741824; do timeout 600 python scripts/r2/inv_odd_probe.py $m 2>&1 | tail -4; done
