set -x
python -c "from paper_1708_07853_b200 import _build; _build.build_variant('tuning', {'DWT2_TUNING': 1})"
for tq in 4096 16384 65536; do
  for llq in 262144 1048576; do
    DWT2_TAIL_QUADS=$tq LLQ=$llq timeout 600 python scripts/r2/small_probe.py 65536 2>&1 | grep 'config 4' | sed "s/^/tail=$tq llq=$llq /"
  done
done
