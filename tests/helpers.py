"""Comparison helpers for GPU-vs-oracle parity (tests only)."""
from __future__ import annotations

import itertools

import numpy as np

FIELDS = ["model", "cut", "K", "cls", "batch", "reserved", "e2e_us", "stage_us"]


def rows_of(points):
    return [tuple(np.asarray(p[f]).tolist() if np.ndim(p[f]) else int(p[f]) for f in FIELDS) for p in points]


def assert_same_points(got, exp, label=""):
    """Element-by-element equality of two 32-byte point arrays (bit-exact)."""
    assert got.dtype.itemsize == 32 and exp.dtype.itemsize == 32
    g = np.frombuffer(np.ascontiguousarray(got).tobytes(), dtype=np.uint32).reshape(-1, 8)
    e = np.frombuffer(np.ascontiguousarray(exp).tobytes(), dtype=np.uint32).reshape(-1, 8)
    if g.shape == e.shape and np.array_equal(g, e):
        return
    n = min(len(g), len(e))
    bad = np.nonzero((g[:n] != e[:n]).any(axis=1))[0]
    i = int(bad[0]) if len(bad) else n
    msg = f"{label}: {len(g)} points vs oracle {len(e)}; first difference at {i}"
    if i < len(got):
        msg += f"\n  gpu    {rows_of(got[i:i + 1])}"
    if i < len(exp):
        msg += f"\n  oracle {rows_of(exp[i:i + 1])}"
    raise AssertionError(msg)


def assert_same_result(g, o, label=""):
    assert g.n_candidates == o.n_candidates, (label, g.n_candidates, o.n_candidates)
    assert g.n_feasible == o.n_feasible, (label, g.n_feasible, o.n_feasible)
    assert_same_points(g.points, o.points, label)
    assert np.array_equal(g.seg_offsets, o.seg_offsets), label


def seg_key(p):
    return (int(p["model"]), int(p["K"]), tuple(int(c) for c in p["cls"][:int(p["K"])]))


def theta_gt(bp, cp, bq, cq):
    return bp * cq > bq * cp


def reduce_union(points):
    """Frontier of a union of per-shard frontiers (decomposability):
    per segment sort by (E asc, theta desc, b asc, cuts asc) and keep strictly
    increasing theta. Test-side helper for shard-mode checks."""
    import functools
    groups = {}
    for p in points:
        groups.setdefault(seg_key(p), []).append(p)
    out = []
    for key in sorted(groups):
        ps = groups[key]

        def cmp(p, q):
            if int(p["e2e_us"]) != int(q["e2e_us"]):
                return -1 if int(p["e2e_us"]) < int(q["e2e_us"]) else 1
            cp, cq = int(max(p["stage_us"])), int(max(q["stage_us"]))
            bp, bq = int(p["batch"]), int(q["batch"])
            if theta_gt(bp, cp, bq, cq):
                return -1
            if theta_gt(bq, cq, bp, cp):
                return 1
            kp = (bp, int(p["cut"][0]), int(p["cut"][1]))
            kq = (bq, int(q["cut"][0]), int(q["cut"][1]))
            return -1 if kp < kq else (1 if kp > kq else 0)

        ps.sort(key=functools.cmp_to_key(cmp))
        bb, bc = 0, 1
        for p in ps:
            c = int(max(p["stage_us"]))
            if theta_gt(int(p["batch"]), c, bb, bc):
                out.append(p)
                bb, bc = int(p["batch"]), c
    if not out:
        return np.zeros(0, dtype=points.dtype if hasattr(points, "dtype") else None)
    return np.array(out, dtype=out[0].dtype)


def segment_points(points, seg_offsets, s):
    return points[int(seg_offsets[s]):int(seg_offsets[s + 1])]


def seg_index_of(w, m, K, cls):
    C = w.n_classes
    base = 0
    for mm in range(m):
        base += sum(C ** k for k in range(1, min(w.kmax, w.models[mm].n_layers) + 1))
    off = sum(C ** k for k in range(1, K))
    idx = 0
    for c in cls:
        idx = idx * C + c
    return base + off + idx


def all_segments(w, m):
    C, M = w.n_classes, w.models[m].n_layers
    for K in range(1, min(w.kmax, M) + 1):
        for cls in itertools.product(range(C), repeat=K):
            yield K, cls
