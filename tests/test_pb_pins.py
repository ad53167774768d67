"""Pins for the oracle's per-stage batch enumeration (oracle_run_pb; SURVEY.md §8(f)
NEXT-4; App. A.1 of PAPER.md: partition d runs at its own batch b_d, eq. 1.1 summing
p_{ldbij} over b per partition; DESIGN.md §3 readings PB-1..PB-4).

Each test fixes the oracle against something other than itself: the unified-batch
oracle where the two must agree, an independent Fraction-based literal definition
(tests/pareto_brute.py), closed-form counts, a hand-worked plan that only exists with
mixed batches, and the superset property over the unified frontier.
"""
from __future__ import annotations

import itertools
from fractions import Fraction
from math import comb, inf

import numpy as np
import pytest

from oracle import run_oracle, run_oracle_pb
from tests import pareto_brute as pb
from tests.fixtures import make_workload
from tests.test_oracle_pins import seg_points
from workloads import config1, config2, config3, random_tiny


def pts_pb(r, w, m, K, cls):
    return [(tuple(int(b) for b in p["bidx"][:K]), int(p["cut"][0]), int(p["cut"][1]), int(p["e2e_us"]))
            for p in seg_points(r, w, m, K, cls)]


def theta_pb(w, p):
    K = int(p["K"])
    return min(Fraction(int(w.batches[p["bidx"][d]]), int(p["stage_us"][d])) if p["stage_us"][d] else inf
               for d in range(K))


def test_pb_hand_worked_mixed_batch_plan():
    """M = 2, one class, batches {1, 4}, no transfer. Layer 0 is heavy and batches well
    (40 us at b=1, 64 at b=4), layer 1 is light (5, 20). Unified K=2: b=1 gives E = 45,
    theta = 1/40; b=4 gives E = 84, theta = min(4/64, 4/20) = 1/16. Per-stage (4, 1):
    C = (64, 5), E = 69, theta = min(4/64, 1/5) = 1/16 -- the unified b=4 throughput 15 us
    earlier. (1, 4): E = 60, theta = 1/40 loses to (1, 1); (4, 4) = unified b=4 loses to (4, 1)."""
    lat = np.array([[[40, 64], [5, 20]]], dtype=np.uint32)
    w = make_workload([lat], [[0, 0]], 1000, [1, 4], 1000, margin=0, kmax=2)
    r = run_oracle_pb(w)
    assert r.n_candidates == 2 + 4 and r.n_feasible == 6
    assert pts_pb(r, w, 0, 2, (0, 0)) == [((0, 0), 1, 0, 45), ((1, 0), 1, 0, 69)]
    assert pts_pb(r, w, 0, 1, (0,)) == [((0,), 0, 0, 45), ((1,), 0, 0, 84)]
    u = run_oracle(w)
    assert [(int(p["batch"]), int(p["e2e_us"])) for p in seg_points(u, w, 0, 2, (0, 0))] == [(1, 45), (4, 84)]


def test_pb_transfer_uses_the_senders_batch():
    """eq. 1.11: the transfer after partition d is Y_{bj} at partition d's batch. S_0 = 1000 B
    over 8 bit/us: Y = 1000 b us. With stage batches (1, 2) the plan pays Y = 1000 (b_1 = 1)."""
    lat = np.array([[[1, 2], [1, 2]]], dtype=np.uint32)
    w = make_workload([lat], [[1000, 0]], 8, [1, 2], 10**6, margin=0, kmax=2)
    r = run_oracle_pb(w)
    got = {p[0]: p[3] for p in pts_pb(r, w, 0, 2, (0, 0))}
    assert got[(0, 0)] == 1002  # (b_1, b_2) = (1, 1): 1 + 1 + Y(b_1 = 1) = 1000
    cands, _ = pb.enumerate_candidates_pb(w, 0)
    Es = {c["bidx"]: c["E"] for c in cands[(2, (0, 0))]}
    assert Es == {(0, 0): 1002, (0, 1): 1003, (1, 0): 2003, (1, 1): 2004}


@pytest.mark.parametrize("seed", range(30))
def test_pb_single_batch_equals_the_unified_oracle(seed):
    w = random_tiny(300 + seed, max_batches=1, n_models=1 + seed % 2)
    assert w.n_batches == 1
    r, u = run_oracle_pb(w), run_oracle(w)
    assert (r.n_candidates, r.n_feasible) == (u.n_candidates, u.n_feasible)
    assert np.array_equal(r.seg_offsets, u.seg_offsets)
    for a, b in zip(r.points, u.points):
        K = int(a["K"])
        assert (int(a["model"]), int(a["K"]), int(a["e2e_us"])) == (int(b["model"]), int(b["K"]), int(b["e2e_us"]))
        assert list(a["cut"]) == list(b["cut"]) and list(a["cls"]) == list(b["cls"])
        assert list(a["stage_us"]) == list(b["stage_us"])
        assert [int(x) for x in a["bidx"][:K]] == [0] * K


@pytest.mark.parametrize("seed", range(40))
def test_pb_literal_fuzz(seed):
    w = random_tiny(400 + seed, max_layers=6, max_batches=3, n_models=1 + seed % 2)
    r = run_oracle_pb(w, threads=1 + seed % 3)
    n_cand = 0
    for m in range(len(w.models)):
        segs, nc = pb.enumerate_candidates_pb(w, m)
        n_cand += nc
        C, M = w.n_classes, w.models[m].n_layers
        for K in range(1, min(w.kmax, M) + 1):
            for cls in itertools.product(range(C), repeat=K):
                lit = pb.literal_frontier_pb(segs.get((K, cls), []))
                got = seg_points(r, w, m, K, cls)
                assert len(got) == len(lit), (m, K, cls)
                for g, e in zip(got, lit):
                    assert int(g["e2e_us"]) == e["E"]
                    assert tuple(int(x) for x in g["bidx"][:K]) == e["bidx"]
                    assert (int(g["cut"][0]), int(g["cut"][1])) == e["cuts"]
                    assert [int(v) for v in g["stage_us"][:K]] == e["stages"]
    assert r.n_candidates == n_cand


@pytest.mark.parametrize("make", [config1, config2, config3])
def test_pb_closed_form_candidate_count(make):
    w = make()
    r = run_oracle_pb(w)
    C, B = w.n_classes, w.n_batches
    exp = sum(comb(m.n_layers - 1, K - 1) * C ** K * B ** K for m in w.models for K in range(1, min(w.kmax, m.n_layers) + 1))
    assert r.n_candidates == exp


@pytest.mark.parametrize("make", [config1, config3] + [lambda s=s: random_tiny(500 + s, max_batches=3) for s in range(10)])
def test_pb_frontier_covers_the_unified_frontier(make):
    """Unified plans are the per-stage plans with b_1 = .. = b_K, so every unified frontier
    point is matched or beaten (E <=, theta >=) by a per-stage frontier point of its segment;
    K = 1 segments coincide."""
    w = make()
    r, u = run_oracle_pb(w), run_oracle(w)
    assert r.n_feasible >= u.n_feasible
    for s in range(len(u.seg_offsets) - 1):
        up = u.points[int(u.seg_offsets[s]):int(u.seg_offsets[s + 1])]
        rp = r.points[int(r.seg_offsets[s]):int(r.seg_offsets[s + 1])]
        for p in up:
            K = int(p["K"])
            cm = max(int(v) for v in p["stage_us"][:K])
            th = Fraction(int(p["batch"]), cm) if cm else inf
            assert any(int(q["e2e_us"]) <= int(p["e2e_us"]) and theta_pb(w, q) >= th for q in rp), s
        if len(up) and int(up[0]["K"]) == 1:
            assert [int(q["e2e_us"]) for q in rp] == [int(q["e2e_us"]) for q in up]
