set -x
mkdir -p gpurun_out/small
python -c "from paper_1708_07853_b200 import _build; _build.build_variant('tuning', {'DWT2_TUNING': 1})"
timeout 300 python __graft_entry__.py smoke
timeout 900 python -m pytest tests/test_gpu_small.py -q -x 2>&1 | tail -3
for m in product 0 262144; do timeout 600 python scripts/r2/small_probe.py $m 2>&1 | tail -5; done
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for c in 1 4; do timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/small/fwd53_c$c.json 2>&1; tail -c 150 gpurun_out/small/fwd53_c$c.json; echo; done
