set -x
timeout 600 python scripts/level_costs.py 8192 8192 8 cdf97 2>&1 | tail -8
timeout 600 python scripts/level_costs.py 8192 8192 8 cdf53 2>&1 | tail -8
