set -x
python -c "from paper_1708_07853_b200 import _build; _build.build_variant('tuning', {'DWT2_TUNING': 1})"
for m in nodf from0 from1 from2 from3; do timeout 600 python scripts/r2/df_probe.py $m 2>&1 | tail -5; done
