set -x
python -c "from paper_1708_07853_b200 import _build; _build.build_variant('tuning', {'DWT2_TUNING': 1})"
for tq in 65536 16384 4096; do DWT2_K2_TAIL_QUADS=$tq timeout 600 python scripts/r2/k2small_probe.py 262144 2>&1 | grep 'config 4' | sed "s/^/tail=$tq /"; done
for tq in 65536 16384; do DWT2_TAIL_QUADS=$tq timeout 600 python scripts/r2/small_probe.py 65536 2>&1 | grep 'config 4' | sed "s/^/53tail=$tq /"; done
