"""Build libppipe_b200.so in-tree with nvcc for sm_100a (B200).

Each source compiles to its own object in parallel (no device code crosses
files), then one nvcc link produces the shared library.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libppipe_b200.so")
SOURCES = [os.path.join(CSRC, f) for f in
           ("ppipe_kernels.cu", "ppipe_f2.cu", "ppipe_pb.cu", "ppipe_frontier.cu", "ppipe_abi.cpp")]
HEADERS = [os.path.join(CSRC, "ppipe_internal.h"), os.path.join(CSRC, "ppipe_block.cuh"), os.path.join(ROOT, "include", "ppipe.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _common(extra=()):
    return ["-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xptxas", "-v", "--expt-relaxed-constexpr",
            "-Xcompiler", "-fPIC,-fvisibility=hidden,-O3", "-I", os.path.join(ROOT, "include"), *extra]


def nvcc_cmd(out: str = LIB, extra=()):
    """Single-invocation form (used by scripts/variants.py for experiment builds)."""
    return [NVCC, *_common(extra), "-shared", "-o", out, *SOURCES, "-ldl"]


def source_hash(extra=()) -> str:
    import hashlib
    h = hashlib.sha256()
    for path in SOURCES + HEADERS:
        with open(path, "rb") as f:
            h.update(f.read())
    h.update(" ".join(nvcc_cmd(extra=extra)).encode())
    return h.hexdigest()


STAMP = LIB + ".stamp"


def stale(lib: str = LIB) -> bool:
    """Content-hash check (snapshot copies need not preserve mtimes)."""
    if not os.path.exists(lib) or not os.path.exists(STAMP):
        return True
    with open(STAMP) as f:
        return f.read().strip() != source_hash()


def build_lib(out: str, extra=(), log_path=None) -> None:
    objdir = os.path.join(os.path.dirname(out), "build", os.path.basename(out) + ".objs")
    os.makedirs(objdir, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        r = subprocess.run([NVCC, *_common(extra), "-c", "-o", obj, src], capture_output=True, text=True)
        return src, obj, r

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    logs = []
    for src, obj, r in results:
        logs.append(r.stdout + r.stderr)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {os.path.basename(src)}")
    r = subprocess.run([NVCC, *ARCH, "-shared", "-o", out, *[o for _, o, _ in results], "-ldl"],
                       capture_output=True, text=True)
    logs.append(r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    if log_path:
        with open(log_path, "w") as f:
            f.write("".join(logs))


def build(force: bool = False, verbose: bool = False) -> str:
    if force or stale():
        log = os.path.join(PKG, "build_ptxas.log")
        build_lib(LIB, log_path=log)
        with open(STAMP, "w") as f:
            f.write(source_hash())
        if verbose:
            sys.stdout.write(open(log).read())
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
