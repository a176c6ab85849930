"""Library selection of the measurement scripts (never the product path).

The binding always loads the in-tree product library.  A script run with
DWT2_LIB=<path> loads that build instead -- e.g. a -DDWT2_PROF build, or
build/variants/libdwt2_tuning.so from
``_build.build_variant("tuning", {"DWT2_TUNING": 1})``, the only build that
reads the DWT2_* tile-policy knobs from the environment.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1708_07853_b200 import dwt2  # noqa: E402

if os.environ.get("DWT2_LIB"):
    dwt2.use_variant(os.environ["DWT2_LIB"])
