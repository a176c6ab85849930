set -x
python -c "from paper_1708_07853_b200 import _build; _build.build_variant('tuning', {'DWT2_TUNING': 1})"
for i in 1 2; do
timeout 300 python bench.py --config 1 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench product c1', d['ms_per_step']*1e3, 'us', d.get('warm_l2'))"
DWT2_SMALL_QUADS=0 timeout 300 python bench.py --config 1 --no-e2e --no-cpu-baseline --variant-lib build/variants/libdwt2_tuning.so 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench levelkernel c1', d['ms_per_step']*1e3, 'us', d.get('warm_l2'))"
done
for m in product 0; do timeout 600 python scripts/r2/small_probe.py $m 2>&1 | tail -5; done
