"""Compile the CUDA library in-tree for sm_100a (used by __graft_entry__.build()).

nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -shared -Xcompiler -fPIC
  csrc/{dwt2,inverse,schemes,dwt97}.cu -> paper_1708_07853_b200/libdwt2.so   (links only cudart; the TMA
descriptor encoder is fetched from the driver at run time).
"""
from __future__ import annotations

import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
SRCS = [os.path.join(PKG, "csrc", f) for f in ("dwt2.cu", "inverse.cu", "schemes.cu", "dwt97.cu", "tail.cu", "peer.cu")]
# every source and header under csrc/ (an edit to any of them rebuilds the library)
DEPS = sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")) + glob.glob(os.path.join(PKG, "csrc", "*.h")) +
              glob.glob(os.path.join(PKG, "csrc", "*.cuh")))
HDR = os.path.join(ROOT, "include", "dwt2.h")
LIB = os.path.join(PKG, "libdwt2.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
    "-Xptxas", "-v", "-cudart", "shared",
]


def build_variant(name: str, defines: dict) -> str:
    """Tuning builds (e.g. stages / warps per CTA) under build/variants/."""
    out_dir = os.path.join(ROOT, "build", "variants")
    os.makedirs(out_dir, exist_ok=True)
    out = os.path.join(out_dir, f"libdwt2_{name}.so")
    cmd = [NVCC, *NVCC_FLAGS, *[f"-D{k}={v}" for k, v in defines.items()], *SRCS, "-o", out]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
    return out


def build(force: bool = False, verbose: bool = False) -> str:
    stale = (not os.path.exists(LIB) or
             os.path.getmtime(LIB) < max([os.path.getmtime(f) for f in DEPS] + [os.path.getmtime(HDR)]))
    if force or stale:
        tmp = LIB + f".tmp{os.getpid()}"
        cmd = [NVCC, *NVCC_FLAGS, *SRCS, "-o", tmp]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
        if verbose:
            print(res.stdout + res.stderr)
        with open(os.path.join(PKG, "csrc", "ptxas_info.txt"), "w") as f:
            f.write(res.stderr)
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose=True)
