set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 120 python __graft_entry__.py smoke 2>&1 | tail -5
timeout 600 python -m pytest tests -m gpu -x -q -k "tiny or config1 or ragged or errors or host" 2>&1 | tail -30
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -5
