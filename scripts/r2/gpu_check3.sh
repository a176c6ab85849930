mkdir -p gpurun_out/r2l
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python scripts/level_costs.py 8192 8192 8 cdf53 inverse 2>&1 | tail -1
timeout 300 python scripts/level_costs.py 8192 8192 8 cdf97 inverse 2>&1 | tail -1
timeout 300 python scripts/level_costs.py 8192 8192 8 cdf97 2>&1 | tail -1
