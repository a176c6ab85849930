"""B200-native forward 2-D CDF 5/3 DWT (non-separable lifting, arXiv:1708.07853).

Public surface: the C ABI in include/dwt2.h (libdwt2.so, built for sm_100a)
and its thin Python binding :mod:`paper_1708_07853_b200.dwt2`.
"""
from . import dwt2  # noqa: F401
from .dwt2 import Plan, StripPlan, forward  # noqa: F401

__all__ = ["dwt2", "Plan", "StripPlan", "forward"]
