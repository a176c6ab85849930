set -x
python -c "from paper_1708_07853_b200 import _build; _build.build_variant('tuning', {'DWT2_TUNING': 1})"
timeout 600 python scripts/r2/small_probe.py product mid 2>&1 | tail -5
timeout 600 python scripts/r2/small_probe.py 100000000 mid 2>&1 | tail -5
LLQ=100000000 timeout 600 python scripts/r2/small_probe.py 100000000 mid 2>&1 | tail -5
