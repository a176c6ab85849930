# GPU check: tests, smoke, bench on every config (one JSON line each)
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -6
timeout 120 python __graft_entry__.py smoke 2>&1 | tail -3
for c in 3 1 2 4 4b 5; do
  timeout 600 python bench.py --config $c > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; tail -1 gpurun_out/bench_c$c.json
done
