"""CPU checks of bench.py's measurement protocol (no GPU): which workloads
count as L2-sized, how many buffer pairs the timed steps cycle over, and that
the JSON config says so."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_1708_07853_b200 import workloads  # noqa: E402

L2 = 126e6


@pytest.mark.parametrize("name", ["1", "2", "3", "4", "4b", "5"])
@pytest.mark.parametrize("steps", [3, 20, 100])
def test_buffer_pairs_keep_every_step_cold(name, steps):
    cfg = workloads.CONFIGS[name]
    pair_bytes = cfg.pixels * 8
    n = bench.buffer_pairs(cfg, steps)
    assert 1 <= n <= max(1, steps)
    if pair_bytes >= 2 * L2:
        assert n == 1                      # inputs larger than the L2: one pair
    elif n < steps:
        # a pair is reused only after more than 2x L2 of other steps' traffic
        assert (n - 1) * pair_bytes > 2 * L2
    else:
        assert n == steps                  # every step its own pair (read once after the flush)
    l2 = bench.describe(cfg, 1, steps)["l2"]
    if pair_bytes < 2 * L2:
        assert f"cycle over {n} input/output pairs" in l2
    else:
        assert "larger than the 126 MB L2" in l2


def test_small_configs_flagged():
    assert bench.buffer_pairs(workloads.CONFIGS["1"], 20) == 20
    assert bench.buffer_pairs(workloads.CONFIGS["2"], 20) == 3
    assert bench.buffer_pairs(workloads.CONFIGS["3"], 20) == 1
