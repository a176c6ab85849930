"""The C ABI used from plain C (examples/forward_c.c): it compiles and links
against libdwt2.so and the CUDA runtime with gcc alone (CPU test), and on a
B200 the ramp image comes out with zero interior details, the ramp in the
coarsest LL and an exact inverse (GPU test)."""
import os
import subprocess

import pytest

from paper_1708_07853_b200 import _build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1708_07853_b200")


def build_example(tmp_path):
    _build.build()
    exe = str(tmp_path / "forward_c")
    cmd = ["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(ROOT, "examples", "forward_c.c"), "-L", PKG, "-ldwt2", "-L", "/usr/local/cuda/lib64",
           "-lcudart", f"-Wl,-rpath,{PKG}", "-lm", "-o", exe]
    res = subprocess.run(cmd, capture_output=True, text=True)
    assert res.returncode == 0, res.stdout + res.stderr
    return exe


def test_c_example_builds(tmp_path):
    assert os.path.exists(build_example(tmp_path))


@pytest.mark.gpu
@pytest.mark.parametrize("W,H,L", [(1000, 777, 3), (4096, 4096, 5), (8193, 301, 4)])
def test_c_example_runs(tmp_path, W, H, L):
    exe = build_example(tmp_path)
    res = subprocess.run([exe, str(W), str(H), str(L)], capture_output=True, text=True, timeout=120)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "max |detail| 0," in res.stdout


def build_peer_example(tmp_path):
    _build.build()
    exe = str(tmp_path / "peer_strips_c")
    cmd = ["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(ROOT, "examples", "peer_strips_c.c"), "-L", PKG, "-ldwt2", "-L", "/usr/local/cuda/lib64",
           "-lcudart", f"-Wl,-rpath,{PKG}", "-o", exe]
    res = subprocess.run(cmd, capture_output=True, text=True)
    assert res.returncode == 0, res.stdout + res.stderr
    return exe


def test_c_peer_example_builds(tmp_path):
    """The peer-strip entry points from plain C (examples/peer_strips_c.c)."""
    assert os.path.exists(build_peer_example(tmp_path))


@pytest.mark.gpu
@pytest.mark.parametrize("W,H,L,G", [(1000, 1024, 3, 4), (777, 513, 2, 3), (4096, 4096, 6, 8)])
def test_c_peer_example_runs(tmp_path, W, H, L, G):
    exe = build_peer_example(tmp_path)
    res = subprocess.run([exe, str(W), str(H), str(L), str(G)], capture_output=True, text=True, timeout=120)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "single-image transform 0" in res.stdout
