"""A larger run of tests/test_gpu_fuzz.py's randomised cases with other seeds
(1500 5/3, 300 CDF 9/7, 150 row-strip pyramids): python scripts/fuzz_many.py.
Last run on B200: all pass."""
import sys, traceback
sys.path.insert(0, '.')
import tests.test_gpu_fuzz as F
bad = 0
cs = F.cases(1500, 4242)
for i, c in enumerate(cs):
    try:
        F.test_forward_inverse_random(*c)
    except AssertionError as e:
        bad += 1
        print("FAIL", c, str(e)[:200])
        if bad > 5: break
print("5/3 cases", len(cs), "bad", bad)
bad = 0
cs = F.cases(300, 777)
for c in cs:
    try:
        F.test_cdf97_random(*c)
    except AssertionError as e:
        bad += 1; print("FAIL97", c, str(e)[:200])
        if bad > 5: break
print("9/7 cases", len(cs), "bad", bad)
bad = 0
cs = F.strip_cases(150, 999)
for c in cs:
    try:
        F.test_strip_pyramids_random(*c)
    except AssertionError as e:
        bad += 1; print("FAILSTRIP", c, str(e)[:200])
        if bad > 5: break
print("strip cases", len(cs), "bad", bad)
