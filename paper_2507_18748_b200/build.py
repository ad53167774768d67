"""Build libppipe_b200.so in-tree with nvcc for sm_100a (B200)."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libppipe_b200.so")
SOURCES = [os.path.join(CSRC, "ppipe_kernels.cu"), os.path.join(CSRC, "ppipe_f2.cu"), os.path.join(CSRC, "ppipe_pb.cu"), os.path.join(CSRC, "ppipe_abi.cpp")]
HEADERS = [os.path.join(CSRC, "ppipe_internal.h"), os.path.join(ROOT, "include", "ppipe.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc_cmd(out: str = LIB, extra=()):
    return [NVCC, "-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xptxas", "-v", "--expt-relaxed-constexpr",
            "-Xcompiler", "-fPIC,-fvisibility=hidden,-O3", "-shared", "-I", os.path.join(ROOT, "include"),
            "-o", out, *SOURCES, "-ldl", *extra]


def source_hash() -> str:
    import hashlib
    h = hashlib.sha256()
    for path in SOURCES + HEADERS:
        with open(path, "rb") as f:
            h.update(f.read())
    h.update(" ".join(nvcc_cmd()).encode())
    return h.hexdigest()


STAMP = LIB + ".stamp"


def stale(lib: str = LIB) -> bool:
    """Content-hash check (snapshot copies need not preserve mtimes)."""
    if not os.path.exists(lib) or not os.path.exists(STAMP):
        return True
    with open(STAMP) as f:
        return f.read().strip() != source_hash()


def build(force: bool = False, verbose: bool = False) -> str:
    if force or stale():
        cmd = nvcc_cmd()
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed building libppipe_b200.so")
        with open(STAMP, "w") as f:
            f.write(source_hash())
        log = os.path.join(PKG, "build_ptxas.log")
        with open(log, "w") as f:
            f.write(r.stdout + r.stderr)
        if verbose:
            sys.stdout.write(r.stderr)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
