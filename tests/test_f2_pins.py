"""Pins for the oracle's F2 reduction (DESIGN.md §3 F2-1..F2-4).

F2 keeps, per segment (model, K, class tuple), the feasible candidates whose
per-stage per-GPU throughput vector x = (b / C_1, .., b / C_K) (X_{ldbij},
PAPER.md:2245) is not dominated, with E as the tie-break only. That is the
candidate set PPipe's pooled MILP can pick from without loss: the pipeline's
throughput is min_d g_d X_d for the GPU counts g it assigns (eqs. 1.10, 1.13,
PAPER.md:2281, 2284), and E only has to meet the SLO (eq. 1.12).

Each test fixes the oracle against something other than itself: hand-worked
fixtures, an independent Fraction-based literal definition
(tests/pareto_brute.py), the K = 1 closed form, a provable all-kept case, and
the losslessness property the frontier exists for.
"""
from __future__ import annotations

import itertools
import math
from fractions import Fraction

import numpy as np
import pytest

from oracle import run_oracle
from tests import pareto_brute as pb
from tests.fixtures import make_workload
from tests.test_oracle_pins import seg_points
from workloads import config1, config2, config3, random_tiny


def pts(r, w, m, K, cls):
    return [(int(p["cut"][0]), int(p["cut"][1]), int(p["batch"]), int(p["e2e_us"])) for p in seg_points(r, w, m, K, cls)]


# ---------------- hand-worked fixtures ----------------

def test_f2_hand_worked_equal_vectors_keep_min_e(oracle_built):
    """M = 2, one class, b in {1, 2}, lat(b=2) = 2 lat(b=1) = (4, 8), S_0 = 125 B over 1000 bit/us
    -> Y = b us. K=1: x = 1/6 at b=1 (E=6) and 2/12 at b=2 (E=12): equal, E decides -> b=1.
    K=2 (c=1): C = (2, 4), E = 7 at b=1; C = (4, 8), E = 14 at b=2: x = (1/2, 1/4) both -> b=1."""
    lat = np.array([[[2, 4], [4, 8]]], dtype=np.uint32)
    w = make_workload([lat], [[125, 0]], 1000, [1, 2], 1000, margin=0, kmax=2)
    r = run_oracle(w, frontier=2)
    assert r.n_feasible == 4
    assert pts(r, w, 0, 1, (0,)) == [(0, 0, 1, 6)]
    assert pts(r, w, 0, 2, (0, 0)) == [(1, 0, 1, 7)]


def test_f2_hand_worked_keeps_incomparable_cuts(oracle_built):
    """M = 3 layers of 1, 2, 3 us, one class, b = 1, no transfer. K=2: c=1 gives C = (1, 5),
    c=2 gives C = (3, 3); x = (1, 1/5) vs (1/3, 1/3) are incomparable -> both stay under F2,
    while the (E, theta) staircase (both E = 6) keeps only c=2 (theta 1/3 > 1/5)."""
    w = make_workload([[[1, 2, 3]]], [[0, 0, 0]], 1000, [1], 1000, margin=0, kmax=2)
    assert pts(run_oracle(w, frontier=2), w, 0, 2, (0, 0)) == [(1, 0, 1, 6), (2, 0, 1, 6)]
    assert pts(run_oracle(w), w, 0, 2, (0, 0)) == [(2, 0, 1, 6)]


@pytest.mark.parametrize("slo,k1,k2", [(1000, [(0, 0, 2, 36)], [(1, 0, 2, 36), (2, 0, 2, 36)]),
                                       (35, [(0, 0, 1, 30)], [(1, 0, 1, 30), (2, 0, 1, 30)])])
def test_f2_hand_worked_cross_batch_dominance(oracle_built, slo, k1, k2):
    """M = 3, one class, b in {1, 2}: lat(b=1) = 10 us per layer, lat(b=2) = 12 us per layer,
    no transfer. K=2: (c=1, b=1) x = (1/10, 1/20) is dominated by (c=1, b=2) x = (1/6, 1/12);
    (c=2, b=1) x = (1/20, 1/10) by (c=2, b=2) x = (1/12, 1/6). K=1: 1/30 < 2/36. With T = 35
    the b = 2 plans (E = 36) are infeasible and the b = 1 plans come back."""
    lat = np.array([[[10, 12], [10, 12], [10, 12]]], dtype=np.uint32)
    w = make_workload([lat], [[0, 0, 0]], 1000, [1, 2], slo, margin=0, kmax=2)
    r = run_oracle(w, frontier=2)
    assert pts(r, w, 0, 1, (0,)) == k1
    assert pts(r, w, 0, 2, (0, 0)) == k2


# ---------------- literal definition (Fractions, independent code) ----------------

def compare_f2_with_literal(w, r, use_np=False, vgpu=None):
    n_cand = 0
    for m in range(len(w.models)):
        segs, nc = pb.enumerate_candidates(w, m)
        n_cand += nc
        C, M = w.n_classes, w.models[m].n_layers
        for K in range(1, min(w.kmax, M) + 1):
            for cls in itertools.product(range(C), repeat=K):
                cands = segs.get((K, cls), [])
                lit = (pb.literal_f2_np if use_np else pb.literal_f2)(cands, cls, vgpu)
                got = seg_points(r, w, m, K, cls)
                assert len(got) == len(lit), (m, K, cls, len(got), len(lit))
                for g, e in zip(got, lit):
                    assert (int(g["batch"]), int(g["cut"][0]), int(g["cut"][1])) == (e["b"],) + e["cuts"]
                    assert int(g["e2e_us"]) == e["E"]
                    assert [int(v) for v in g["stage_us"][:K]] == e["stages"]
                    assert list(g["cls"][:K]) == list(cls) and int(g["K"]) == K and int(g["model"]) == m
    assert r.n_candidates == n_cand


@pytest.mark.parametrize("seed", range(60))
def test_f2_literal_fuzz(oracle_built, seed):
    w = random_tiny(seed, n_models=1 + seed % 2)
    compare_f2_with_literal(w, run_oracle(w, threads=1 + seed % 3, frontier=2))


def test_f2_literal_config1(oracle_built):
    w = config1()
    compare_f2_with_literal(w, run_oracle(w, frontier=2))


@pytest.mark.slow
def test_f2_literal_config2(oracle_built):
    w = config2()
    compare_f2_with_literal(w, run_oracle(w, frontier=2), use_np=True)


# ---------------- closed forms ----------------

@pytest.mark.parametrize("make", [config1, config2, config3] + [lambda s=s: random_tiny(100 + s, n_models=2)
                                                               for s in range(20)])
def test_f2_k1_closed_form(oracle_built, make):
    """K = 1 has one stage: x = b / C(b) with C(b) the whole-model latency. The F2 point of
    segment (k) is the feasible batch with the largest b / C, ties to the smaller C (= E),
    then the smaller b -- computed here from the raw profile sums."""
    w = make()
    r = run_oracle(w, frontier=2)
    for m, mp in enumerate(w.models):
        T = pb.t_eff(w.slo_us[m], w.margin_permille)
        for k in range(w.n_classes):
            tot = [int(mp.lat_us[k, :, bi].astype(np.int64).sum()) for bi in range(w.n_batches)]
            feas = [(int(w.batches[bi]), tot[bi]) for bi in range(w.n_batches) if tot[bi] <= T]
            exp = []
            if feas:
                best = max(feas, key=lambda bc: (Fraction(bc[0], bc[1]) if bc[1] else math.inf, -bc[1], -bc[0]))
                exp = [(0, 0, best[0], best[1])]
            assert pts(r, w, m, 1, (k,)) == exp, (m, k)


@pytest.mark.parametrize("seed", range(12))
def test_f2_single_batch_positive_latency_keeps_all(oracle_built, seed):
    """One batch and every layer > 0 us: for two cut sets of one segment, moving a cut
    left shrinks one stage and grows its neighbour strictly, so no two candidates are
    comparable and every feasible candidate is an F2 point (K >= 2). Counted here by
    direct enumeration."""
    rng = np.random.default_rng(seed)
    C, M = int(rng.integers(1, 4)), int(rng.integers(3, 13))
    lat = rng.integers(1, 40, size=(C, M, 1)).astype(np.uint32)
    S = (rng.integers(0, 5, size=M) * 500).astype(np.uint64)
    bw = rng.choice([500, 1000, 4000], size=(C, C)).astype(np.uint32)
    tot = int(lat.sum(axis=1).max())
    w = make_workload([lat], [S], bw, [int(rng.integers(1, 9))], int(tot * rng.uniform(0.5, 1.2)) + 1, kmax=3)
    r = run_oracle(w, frontier=2)
    segs, _ = pb.enumerate_candidates(w, 0)
    for K in (2, 3):
        for cls in itertools.product(range(C), repeat=K):
            got = pts(r, w, 0, K, cls)
            exp = sorted((c["cuts"][0], c["cuts"][1], c["b"], c["E"]) for c in segs.get((K, cls), []))
            assert sorted(got) == exp, (K, cls)


# ---------------- properties ----------------

def best_pipeline_throughput(cands, cls, g):
    """max over candidates of min_d g_d X_d (the MILP's pipeline throughput x_l for GPU
    counts g_d per stage)."""
    best = None
    for c in cands:
        x = pb.stage_vector(c, cls)
        val = min(gd * xd for gd, xd in zip(g, x))
        best = val if best is None else max(best, val)
    return best


@pytest.mark.parametrize("seed", range(30))
def test_f2_is_lossless_for_the_pooled_milp(oracle_built, seed):
    """The reason F2 exists: for every GPU-count vector g, the best pipeline throughput over
    the F2 frontier equals the best over all feasible candidates of the segment."""
    w = random_tiny(200 + seed, n_models=1, kmax=3)
    r = run_oracle(w, frontier=2)
    segs, _ = pb.enumerate_candidates(w, 0)
    rng = np.random.default_rng(seed)
    for (K, cls), cands in segs.items():
        fr = [dict(b=int(p["batch"]), stages=[int(v) for v in p["stage_us"][:K]]) for p in seg_points(r, w, 0, K, cls)]
        assert bool(fr) == bool(cands)
        for _ in range(12):
            g = [int(v) for v in rng.integers(1, 7, size=K)]
            assert best_pipeline_throughput(fr, cls, g) == best_pipeline_throughput(cands, cls, g), (K, cls, g)


def test_f2_vgpu_weights_are_neutral(oracle_built):
    """Virtual GPUs scale stage d of every candidate of a segment by the same v_{k_d}, which
    preserves vector dominance: the F2 frontier does not depend on them."""
    for w in (config2(), config3()):
        base = run_oracle(w, frontier=2)
        rng = np.random.default_rng(7)
        v = [int(x) for x in rng.integers(1, 5, size=w.n_classes)]
        r = run_oracle(w, frontier=2, vgpu=v)
        assert np.array_equal(r.points.view(np.uint8), base.points.view(np.uint8))


def test_f2_contains_the_max_theta_of_every_segment(oracle_built):
    """A candidate dominating p in every stage also has min_d X_d >= p's, so the largest
    bottleneck throughput of a segment is attained on F2; it equals the last point of the
    (E, theta) staircase."""
    for w in (config2(), config3()):
        r1, r2 = run_oracle(w), run_oracle(w, frontier=2)
        assert r1.n_feasible == r2.n_feasible and len(r1.seg_offsets) == len(r2.seg_offsets)
        for s in range(len(r1.seg_offsets) - 1):
            a = r1.points[int(r1.seg_offsets[s]):int(r1.seg_offsets[s + 1])]
            b = r2.points[int(r2.seg_offsets[s]):int(r2.seg_offsets[s + 1])]
            assert (len(a) == 0) == (len(b) == 0)
            if len(a):
                def th(p):
                    cm = max(int(v) for v in p["stage_us"][:int(p["K"])])
                    return Fraction(int(p["batch"]), cm) if cm else math.inf
                assert max(th(p) for p in b) == th(a[-1]), s
