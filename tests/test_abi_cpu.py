"""Host-side checks of the C-ABI library that need no GPU: it loads, exports
every symbol include/ppipe.h declares, validates inputs with named errors, fails
loudly (no CPU fallback) when there is no device, and partitions work across
ranks exactly."""
from __future__ import annotations

import ctypes as ct
import os
import re
import subprocess

import numpy as np
import pytest

from tests.conftest import ROOT


@pytest.fixture(scope="module")
def pplib():
    from paper_2507_18748_b200.build import build
    build()
    import paper_2507_18748_b200 as pp
    pp.lib()
    return pp


def header_functions():
    src = open(os.path.join(ROOT, "include", "ppipe.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ppipe_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(pplib):
    names = header_functions()
    assert {"ppipe_load_profiles", "ppipe_enumerate", "ppipe_pareto", "ppipe_free"} <= set(names)
    out = subprocess.check_output(["nm", "-D", "--defined-only", pplib.LIB_PATH], text=True)
    exported = set(re.findall(r"\bT (ppipe_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    L = ct.CDLL(pplib.LIB_PATH)
    for n in names:
        assert hasattr(L, n)


def test_no_internal_symbols_leak(pplib):
    out = subprocess.check_output(["nm", "-D", "--defined-only", pplib.LIB_PATH], text=True)
    funcs = re.findall(r"\bT (\S+)", out)
    assert all(f.startswith("ppipe_") for f in funcs), [f for f in funcs if not f.startswith("ppipe_")][:5]


def test_library_built_for_sm100a(pplib):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", pplib.LIB_PATH], text=True)
    assert "sm_100a" in out


def _load(pp, lat, S, C, batches, bw, **kw):
    return pp.load_profiles([np.asarray(x, dtype=np.uint32) for x in lat], [np.asarray(s, dtype=np.uint64) for s in S],
                            C, np.asarray(batches, dtype=np.uint32), np.asarray(bw, dtype=np.uint32), **kw)


@pytest.mark.parametrize("case,code,needle", [
    ("zero_bw", -1, "bandwidth class 0 -> class 1"),
    ("batches_not_increasing", -1, "strictly increasing"),
    ("batch_zero", -1, "batch 0 value 0"),
    ("too_many_classes", -1, "n_classes 9"),
    ("huge_latency", -2, "model 0 class 1 batch 1"),
    ("huge_act", -2, "model 0 layer 2"),
    ("no_layers", -1, "model 0: n_layers 0"),
])
def test_validation_errors_name_the_item(pplib, case, code, needle):
    pp = pplib
    lat = np.ones((2, 3, 1), np.uint32)
    S = np.zeros(3, np.uint64)
    bw = np.full((2, 2), 100, np.uint32)
    batches = [1]
    C = 2
    if case == "zero_bw":
        bw[0, 1] = 0
    elif case == "batches_not_increasing":
        lat = np.ones((2, 3, 2), np.uint32)
        batches = [2, 2]
    elif case == "batch_zero":
        batches = [0]
    elif case == "too_many_classes":
        C = 9
        lat = np.ones((9, 3, 1), np.uint32)
        bw = np.ones((9, 9), np.uint32)
    elif case == "huge_latency":
        lat[1, :, 0] = 1 << 27
    elif case == "huge_act":
        S[2] = 1 << 62
    elif case == "no_layers":
        lat = np.ones((2, 0, 1), np.uint32)
        S = np.zeros(0, np.uint64)
    with pytest.raises(pp.PPipeError) as e:
        _load(pp, [lat], [S], C, batches, bw)
    assert e.value.code == code
    assert needle in str(e.value)


def test_no_cpu_fallback_without_device(pplib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(pplib.PPipeError) as e:
        _load(pplib, [np.ones((1, 3, 1), np.uint32)], [np.zeros(3)], 1, [1], [[10]])
    assert e.value.code == -4 and "no CPU fallback" in str(e.value)


def test_build_has_no_compiler_warnings(pplib):
    """A warning such as a misplaced '#pragma unroll' silently changes the kernels."""
    import os
    log = os.path.join(os.path.dirname(pplib.LIB_PATH), "build_ptxas.log")
    if not os.path.exists(log):
        pytest.skip("library not built in this checkout")
    bad = [l for l in open(log) if "warning" in l.lower()]
    assert not bad, "".join(bad[:5])


def test_prepartition_validates_before_touching_a_device(pplib):
    lat, S = [np.ones((2, 5, 3), np.uint32)], [np.zeros(5, np.uint64)]
    with pytest.raises(pplib.PPipeError) as e:
        pplib.prepartition(lat, S, 6)
    assert e.value.code == -1 and "n_blocks 6 must be 1..5" in str(e.value)
    with pytest.raises(pplib.PPipeError) as e:
        pplib.prepartition(lat, S, 2, ref_class=2)
    assert e.value.code == -1 and "reference class" in str(e.value)
    import torch
    if not torch.cuda.is_available():
        with pytest.raises(pplib.PPipeError) as e:
            pplib.prepartition(lat, S, 2)
        assert e.value.code == -4 and "no CPU fallback" in str(e.value)


def _weights(Ms, C, B, rows):
    w = 0
    for M, (lo, hi) in zip(Ms, rows):
        for r in range(lo, hi):
            if r == 0:
                w += C * B
            else:
                w += C * C * B + (C ** 3 * B * (M - 1 - r) if r <= M - 2 else 0)
    return w


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_partition_covers_every_row_once_and_balances(pplib, world):
    rng = np.random.default_rng(world)
    Ms = [int(x) for x in rng.integers(1, 900, size=37)]
    C, B = 5, 64
    parts = [pplib.partition_rows(Ms, C, B, 3, r, world) for r in range(world)]
    for m, M in enumerate(Ms):
        covered = []
        for r in range(world):
            lo, hi = parts[r][m]
            covered += list(range(lo, hi))
        assert covered == list(range(M)), m  # contiguous, rank order, exactly once
    total = _weights(Ms, C, B, [(0, M) for M in Ms])
    maxrow = C ** 3 * B * max(Ms) + C * C * B
    for r in range(world):
        wr = _weights(Ms, C, B, parts[r])
        assert abs(wr - total / world) <= maxrow


@pytest.mark.parametrize("fn", ["update_profiles", "update_profiles_async"])
def test_update_rejects_arrays_that_do_not_match_the_context(pplib, fn):
    """The C side copies C*M*B values from the caller's pointer; the binding must
    refuse arrays with fewer classes or batches than the loaded context (EINVAL)
    before any pointer reaches the library."""
    ctx = pplib.Context(None, 1, n_classes=3, n_batches=4)
    for shape in [(2, 5, 4), (3, 5, 2), (3, 5)]:
        with pytest.raises(pplib.PPipeError) as e:
            getattr(pplib, fn)(ctx, [np.ones(shape, np.uint32)], [np.zeros(5, np.uint64)])
        assert e.value.code == -1
