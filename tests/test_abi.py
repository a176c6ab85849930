"""CPU-side checks of the C ABI: the library builds for sm_100a, loads, and
exports every function include/dwt2.h declares (no compute call without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_1708_07853_b200 import _build, dwt2

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dwt2.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(dwt2_[a-z_]+)\s*\(", src)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return dwt2.lib()


def test_header_declares_expected_api():
    names = declared_functions()
    for n in ["dwt2_plan_create", "dwt2_forward", "dwt2_destroy", "dwt2_forward_batched",
              "dwt2_plan_create_strip", "dwt2_forward_strip", "dwt2_forward_host", "dwt2_last_error",
              "dwt2_error_string"]:
        assert n in names


def test_every_declared_symbol_exported(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", dwt2.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (dwt2_\w+)", out))
    for name in declared_functions():
        assert name in exported, name
        assert hasattr(lib, name)
    assert set(dwt2.SIGNATURES) == set(declared_functions())


def test_library_is_sm100a(lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", dwt2.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", dwt2.LIB_PATH],
                          capture_output=True, text=True).stdout
    assert "UTMALDG" in sass          # TMA-staged tile loads
    assert "SHFL" in sass             # warp-shuffle neighbour exchange
    assert "DFMA" in sass             # fp64 register arithmetic


def test_product_library_reads_no_environment(lib):
    """The tile-policy knobs are compiled in only for -DDWT2_TUNING builds
    (dwt2_internal.h tuning_int): the product library's behaviour and timing
    cannot depend on the caller's environment."""
    out = subprocess.run(["nm", "-D", "--undefined-only", dwt2.LIB_PATH], capture_output=True, text=True).stdout
    assert "getenv" not in out and "secure_getenv" not in out


def test_static_strings(lib):
    assert "sm_100a" in dwt2.version()
    assert dwt2.error_string(0) == "ok"
    assert dwt2.error_string(dwt2.DWT2_EINVAL) == "invalid argument"
    assert dwt2.error_string(12345) == "unknown error"


def test_plan_info_struct_layout():
    assert ctypes.sizeof(dwt2.PlanInfo) == 6 * 4 + 2 * 8


def test_oracle_not_imported_by_product():
    pkg = os.path.join(ROOT, "paper_1708_07853_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "dwt53_oracle" not in txt, f


def test_peer_desc_layout_matches_header(tmp_path):
    """dwt2_peer_desc_t crosses process boundaries as raw bytes (all_gather of
    the descriptor): the ctypes mirror must have the C layout exactly."""
    src = tmp_path / "desc.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "dwt2.h"\n'
                   'int main(void) { printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(dwt2_peer_desc_t), '
                   'offsetof(dwt2_peer_desc_t, base), offsetof(dwt2_peer_desc_t, pid), '
                   'offsetof(dwt2_peer_desc_t, row_begin), offsetof(dwt2_peer_desc_t, owned_off), '
                   'offsetof(dwt2_peer_desc_t, flags_off)); return 0; }\n')
    exe = tmp_path / "desc"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    D = dwt2.PeerDesc
    assert got == [ctypes.sizeof(D), D.base.offset, D.pid.offset, D.row_begin.offset, D.owned_off.offset,
                   D.flags_off.offset]
    d = D()
    d.row_begin, d.flags_off = 128, 4096
    assert D.from_bytes(d.to_bytes()).flags_off == 4096
    with pytest.raises(ValueError):
        D.from_bytes(b"\0" * 10)
