"""Literal definitions used to pin the oracle (tests only).

Independent of oracle/ppipe_oracle.c: candidates are enumerated with
itertools straight from the paper's definitions, and the frontier is the
literal O(n^2) non-domination test (SURVEY.md §8(c) pin P8), not a sort+scan.
"""
from __future__ import annotations

import itertools
import math
from fractions import Fraction

import numpy as np


def t_eff(slo_us: int, margin_permille: int) -> int:
    # "deduct ... margin from the SLO", floor to integer us (reading A5)
    return (int(slo_us) * (1000 - int(margin_permille))) // 1000


def enumerate_candidates(w, m: int, slo_us=None, vgpu=None):
    """All candidates of model m: dict segment(K, cls) -> list of candidate dicts.
    vgpu: per-class virtual-GPU counts; a stage on class k with v_k instances per
    physical GPU has per-GPU throughput v_k b / C, the plan
    the minimum over its stages (x_l = min_d x_ld)."""
    mp = w.models[m]
    lat = mp.lat_us.astype(object)
    S = [int(x) for x in mp.act_bytes]
    C, M, B = mp.lat_us.shape
    T = t_eff(w.slo_us[m] if slo_us is None else slo_us, w.margin_permille)
    out = {}
    n_cand = 0
    for K in range(1, min(w.kmax, M) + 1):
        for cuts in itertools.combinations(range(1, M), K - 1):
            bounds = (0,) + cuts + (M,)
            for cls in itertools.product(range(C), repeat=K):
                for bi in range(B):
                    b = int(w.batches[bi])
                    stages = [sum(int(lat[cls[d], l, bi]) for l in range(bounds[d], bounds[d + 1]))
                              for d in range(K)]
                    trans = [-(-8 * S[bounds[d + 1] - 1] * b // int(w.bw[cls[d], cls[d + 1]]))
                             for d in range(K - 1)]
                    E = sum(stages) + sum(trans)
                    n_cand += 1
                    if E > T:
                        continue
                    cand = dict(E=E, b=b, cmax=max(stages), cuts=tuple(cuts) + (0,) * (2 - len(cuts)),
                                stages=stages, trans=trans)
                    if vgpu is not None:
                        cand["theta"] = min(Fraction(int(vgpu[cls[d]]) * b, stages[d]) if stages[d] > 0
                                            else Fraction(10**30) for d in range(K))
                    out.setdefault((K, cls), []).append(cand)
    return out, n_cand


def theta(c):
    if "theta" in c:
        return c["theta"]
    return Fraction(c["b"], c["cmax"]) if c["cmax"] > 0 else Fraction(10**30)


def literal_frontier(cands):
    """Keep p iff no q dominates it: q has E_q <= E_p and theta_q >= theta_p, and either
    is strictly better in one objective, or equal in both and canonically smaller
    (batch, then cuts) -- reading A1 / A17."""
    keep = []
    for p in cands:
        tp = theta(p)
        dominated = False
        for q in cands:
            if q is p:
                continue
            tq = theta(q)
            if q["E"] <= p["E"] and tq >= tp:
                if q["E"] < p["E"] or tq > tp:
                    dominated = True
                    break
                if (q["b"], q["cuts"]) < (p["b"], p["cuts"]):
                    dominated = True
                    break
        if not dominated:
            keep.append(p)
    keep.sort(key=lambda c: c["E"])
    return keep


def literal_frontier_np(cands):
    """Same literal O(n^2) definition, vectorised with numpy for a few thousand points."""
    if not cands:
        return []
    E = np.array([c["E"] for c in cands], dtype=np.int64)
    b = np.array([c["b"] for c in cands], dtype=np.int64)
    cm = np.array([c["cmax"] for c in cands], dtype=np.int64)
    key = np.array([(c["b"] << 32) | (c["cuts"][0] << 16) | c["cuts"][1] for c in cands], dtype=np.int64)
    keep = []
    for i in range(len(cands)):
        # theta_q >= theta_p  <=>  b_q * cm_p >= b_p * cm_q
        ge = b * cm[i] >= b[i] * cm
        gt = b * cm[i] > b[i] * cm
        dom = (E <= E[i]) & ge & ((E < E[i]) | gt | (key < key[i]))
        dom[i] = False
        if not dom.any():
            keep.append(cands[i])
    keep.sort(key=lambda c: c["E"])
    return keep


# ---------------- F2: the MILP-lossless per-stage frontier ----------------

def stage_vector(c, cls, vgpu=None):
    """x = (X_1, .., X_K), X_d = v_{k_d} b / C_d as exact Fractions (per-GPU throughput of
    stage d, PAPER.md:2245 X_{ldbij} = b / C; virtual GPUs PAPER.md:1107-1126); C_d = 0 is +inf."""
    out = []
    for d, C in enumerate(c["stages"]):
        v = 1 if vgpu is None else int(vgpu[cls[d]])
        out.append(Fraction(v * c["b"], C) if C > 0 else math.inf)
    return tuple(out)


def literal_f2(cands, cls, vgpu=None):
    """Keep p iff no feasible q of the segment has x_q >= x_p in every stage and either
    x_q != x_p, or x_q == x_p and (E, b, cuts)_q < (E, b, cuts)_p. Output in (b, cuts) order."""
    xs = [stage_vector(c, cls, vgpu) for c in cands]
    keep = []
    for i, p in enumerate(cands):
        redundant = False
        for j, q in enumerate(cands):
            if j == i:
                continue
            if all(a >= b for a, b in zip(xs[j], xs[i])):
                if xs[j] != xs[i] or (q["E"], q["b"], q["cuts"]) < (p["E"], p["b"], p["cuts"]):
                    redundant = True
                    break
        if not redundant:
            keep.append(p)
    keep.sort(key=lambda c: (c["b"], c["cuts"]))
    return keep


def literal_f2_np(cands, cls, vgpu=None):
    """literal_f2 vectorised with numpy (integer cross-multiplication: X_q,d >= X_p,d iff
    v b_q C_p,d >= v b_p C_q,d; C = 0 is +inf on both sides)."""
    if not cands:
        return []
    K = len(cands[0]["stages"])
    v = np.array([1 if vgpu is None else int(vgpu[cls[d]]) for d in range(K)], dtype=np.int64)
    b = np.array([c["b"] for c in cands], dtype=np.int64)
    st = np.array([c["stages"] for c in cands], dtype=np.int64)
    E = np.array([c["E"] for c in cands], dtype=np.int64)
    rank = np.array([(c["b"] << 32) | (c["cuts"][0] << 16) | c["cuts"][1] for c in cands], dtype=np.int64)
    keep = []
    for i in range(len(cands)):
        lhs = v * b[:, None] * st[i][None, :]   # v b_q C_p
        rhs = v * b[i] * st                      # v b_p C_q
        ge = (lhs >= rhs).all(axis=1)
        eq = (lhs == rhs).all(axis=1)
        tie_better = (E < E[i]) | ((E == E[i]) & (rank < rank[i]))
        red = ge & (~eq | tie_better)
        red[i] = False
        if not red.any():
            keep.append(cands[i])
    keep.sort(key=lambda c: (c["b"], c["cuts"]))
    return keep


# ---------------- per-stage batch sizes (App. A.1) ----------------

def enumerate_candidates_pb(w, m: int):
    """All per-stage-batch candidates of model m: dict (K, cls) -> list of dicts. Partition d
    runs at its own batch b_d (eq. 1.1 sums over b per partition); the
    transfer after partition d uses the sender's batch (Y_{bj}, eq. 1.11)."""
    mp = w.models[m]
    lat = mp.lat_us.astype(object)
    S = [int(x) for x in mp.act_bytes]
    C, M, B = mp.lat_us.shape
    T = t_eff(w.slo_us[m], w.margin_permille)
    out, n_cand = {}, 0
    for K in range(1, min(w.kmax, M) + 1):
        for cuts in itertools.combinations(range(1, M), K - 1):
            bounds = (0,) + cuts + (M,)
            for cls in itertools.product(range(C), repeat=K):
                for bis in itertools.product(range(B), repeat=K):
                    bs = [int(w.batches[bi]) for bi in bis]
                    stages = [sum(int(lat[cls[d], l, bis[d]]) for l in range(bounds[d], bounds[d + 1]))
                              for d in range(K)]
                    trans = [-(-8 * S[bounds[d + 1] - 1] * bs[d] // int(w.bw[cls[d], cls[d + 1]])) for d in range(K - 1)]
                    E = sum(stages) + sum(trans)
                    n_cand += 1
                    if E > T:
                        continue
                    theta = min(Fraction(bs[d], stages[d]) if stages[d] > 0 else math.inf for d in range(K))
                    out.setdefault((K, cls), []).append(dict(E=E, theta=theta, bidx=tuple(bis), stages=stages,
                                                             cuts=tuple(cuts) + (0,) * (2 - len(cuts))))
    return out, n_cand


def literal_frontier_pb(cands):
    """Keep p iff no q has E_q <= E_p and theta_q >= theta_p with one strict, or both equal and
    (b_1..b_K, cuts)_q < (b_1..b_K, cuts)_p. Output in E order."""
    keep = []
    for p in cands:
        dominated = False
        for q in cands:
            if q is p:
                continue
            if q["E"] <= p["E"] and q["theta"] >= p["theta"]:
                if q["E"] < p["E"] or q["theta"] > p["theta"] or (q["bidx"], q["cuts"]) < (p["bidx"], p["cuts"]):
                    dominated = True
                    break
        if not dominated:
            keep.append(p)
    keep.sort(key=lambda c: c["E"])
    return keep
