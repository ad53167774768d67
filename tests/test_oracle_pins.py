"""Pins for the CPU oracle (invariants I1-I8).

Each test fixes the oracle against something other than itself: a hand-worked
fixture, a number the paper prints, a closed form, a textbook routine, or the
literal O(n^2) definition of the Pareto frontier (tests/pareto_brute.py).
"""
from __future__ import annotations

import itertools
import math
from fractions import Fraction

import numpy as np
import pytest

from oracle import run_oracle
from tests.fixtures import MIB, make_workload, t0, t1
from tests import pareto_brute as pb
from workloads import config1, config2, config3, random_tiny


def seg_index(C, kmax, M, K, cls):
    off = sum(C ** k for k in range(1, K))
    idx = 0
    for c in cls:
        idx = idx * C + c
    return off + idx


def seg_points(res, w, m, K, cls):
    C = w.n_classes
    base = 0
    for mm in range(m):
        base += sum(C ** k for k in range(1, min(w.kmax, w.models[mm].n_layers) + 1))
    s = base + seg_index(C, w.kmax, w.models[m].n_layers, K, cls)
    return res.points[int(res.seg_offsets[s]):int(res.seg_offsets[s + 1])]


def tup(p):
    return (int(p["cut"][0]), int(p["batch"]), int(p["e2e_us"]))


# ---------------- P0a / P0b: hand-worked fixtures ----------------

def test_p0a_hand_worked_t0(oracle_built):
    w = t0()
    r = run_oracle(w)
    assert r.n_candidates == 6 and r.n_feasible == 6
    k1 = seg_points(r, w, 0, 1, (0,))
    assert [(int(p["batch"]), int(p["e2e_us"])) for p in k1] == [(1, 90), (2, 160)]
    k2 = seg_points(r, w, 0, 2, (0, 0))
    # (c=2,b=1,E=92), (c=1,b=1,E=98), (c=2,b=2,E=164); (c=1,b=2) dominated by (c=2,b=2)
    assert [tup(p) for p in k2] == [(2, 1, 92), (1, 1, 98), (2, 2, 164)]
    st = {tup(p): list(p["stage_us"][:2]) for p in k2}
    assert st[(2, 1, 92)] == [60, 30] and st[(1, 1, 98)] == [40, 50] and st[(2, 2, 164)] == [90, 70]


@pytest.mark.parametrize("slo,exp1,exp2", [(100, [(1, 90)], [(2, 1, 92), (1, 1, 98)]),
                                            (95, [(1, 90)], [(2, 1, 92)])])
def test_p0a_slo_prefix(oracle_built, slo, exp1, exp2):
    w = t0(slo)
    r = run_oracle(w)
    assert [(int(p["batch"]), int(p["e2e_us"])) for p in seg_points(r, w, 0, 1, (0,))] == exp1
    assert [tup(p) for p in seg_points(r, w, 0, 2, (0, 0))] == exp2


def test_p0b_tie_break_canonical_cut(oracle_built):
    w = t1()
    r = run_oracle(w)
    k2 = seg_points(r, w, 0, 2, (0, 0))
    assert [tup(p) for p in k2] == [(1, 1, 20)]
    assert [(int(p["batch"]), int(p["e2e_us"])) for p in seg_points(r, w, 0, 1, (0,))] == [(1, 20)]


# ---------------- P1-P4: numbers printed in the paper ----------------

def test_p1_v100_bs2_162_req_per_s(oracle_built):
    # V100, batch 2, 12.3 ms -> (2 x 1 / 0.0123) = 162 req/s; SLO 33.3 ms, 40% margin.
    w = make_workload([np.array([6660, 12300], dtype=np.uint32).reshape(1, 1, 2)], [[0]], 10000, [1, 2], 33300,
                      margin=400, kmax=1)
    r = run_oracle(w)
    pts = seg_points(r, w, 0, 1, (0,))
    last = pts[-1]
    assert int(last["batch"]) == 2 and int(last["stage_us"][0]) == 12300
    assert 12300 <= (33300 * 600) // 1000 == 19980
    req_s = Fraction(int(last["batch"]) * 10**6, int(last["stage_us"][0]))
    assert round(float(req_s), 1) == 162.6 and int(req_s) == 162


def test_p2_fcn_two_pool_plan(oracle_built):
    # P4 pool (12 GPUs) then half-V100 pool (6 vGPUs), bs 1, 1.4 ms transfer;
    # pool throughputs 1082 and 1050 req/s. Blocks: P4 11,091 us, half-V100 5,714 us (DESIGN.md pins).
    lat = np.zeros((2, 2, 1), dtype=np.uint32)
    lat[0, :, 0] = [11091, 30000]   # class 0 = P4
    lat[1, :, 0] = [30000, 5714]    # class 1 = half V100
    w = make_workload([lat], [[1750000, 0]], 10000, [1], 33300, margin=400, kmax=2)
    r = run_oracle(w)
    pts = seg_points(r, w, 0, 2, (0, 1))
    assert len(pts) == 1
    p = pts[0]
    c1, c2 = int(p["stage_us"][0]), int(p["stage_us"][1])
    assert (c1, c2) == (11091, 5714)
    assert int(p["e2e_us"]) - c1 - c2 == 1400  # ceil(8 * 1.75e6 / 1e4) us
    assert int(p["e2e_us"]) == 18205 <= 19980
    assert round(12 * 10**6 / c1) == 1082 and int(6 * 10**6 / c2) == 1050


def test_p3_one_tenth_on_low_class_is_1_9x(oracle_built):
    # high class 10x faster; 1/10 of the layers on the low class -> 1.9x latency.
    lat = np.zeros((2, 10, 1), dtype=np.uint32)
    lat[0, :, 0] = 1000    # high
    lat[1, :, 0] = 10000   # low
    w = make_workload([lat], [[0] * 10], 10000, [1], 10**6, margin=0, kmax=2)
    r = run_oracle(w)
    high = seg_points(r, w, 0, 1, (0,))
    mixed = seg_points(r, w, 0, 2, (1, 0))
    assert int(high[0]["e2e_us"]) == 10000
    assert [(int(p["cut"][0]), int(p["e2e_us"])) for p in mixed] == [(1, 19000)]
    assert Fraction(int(mixed[0]["e2e_us"]), int(high[0]["e2e_us"])) == Fraction(19, 10)


@pytest.mark.parametrize("S,bw,expect_us", [
    (3 * MIB, 32000, 787),      # PAPER.md:734-736 "3 MB ... 0.8 ms" at 32 Gbps
    (50 * MIB, 32000, 13108),   # "50 MB ... 13.2 ms" (MiB reading A4: 13.1 ms, ceil)
    (6375000, 10000, 5100),     # PAPER.md:1888-1889 "5.1 ms" at 10 Gbps effective
])
def test_p4_transfer_pins(oracle_built, S, bw, expect_us):
    w = make_workload([[[1, 1]]], [[S, 0]], bw, [1], 10**7, margin=0, kmax=2)
    r = run_oracle(w)
    p = seg_points(r, w, 0, 2, (0, 0))[0]
    assert int(p["e2e_us"]) - int(p["stage_us"][0]) - int(p["stage_us"][1]) == expect_us


# ---------------- P5, P9: closed forms ----------------

@pytest.mark.parametrize("C,kmax,nseg", [(2, 3, 14), (2, 2, 6), (3, 3, 39), (4, 3, 84), (5, 3, 155)])
def test_p5_segment_counts(oracle_built, C, kmax, nseg):
    lat = np.ones((C, 4, 1), dtype=np.uint32)
    w = make_workload([lat], [[0] * 4], 1000, [1], 10**6, kmax=kmax)
    r = run_oracle(w)
    assert len(r.seg_offsets) - 1 == nseg


def closed_form_count(w):
    C, B = w.n_classes, w.n_batches
    return sum(math.comb(mp.n_layers - 1, K - 1) * C ** K * B
               for mp in w.models for K in range(1, min(w.kmax, mp.n_layers) + 1))


@pytest.mark.parametrize("cfg,expect", [(config1, 90), (config2, 122496), (config3, 1412352)])
def test_p9_candidate_count(oracle_built, cfg, expect):
    w = cfg()
    assert closed_form_count(w) == expect
    assert run_oracle(w).n_candidates == expect


# ---------------- P6: K=1 closed form ----------------

@pytest.mark.parametrize("cfg", [config2, config3])
def test_p6_k1_plain_batched_latency_bound(oracle_built, cfg):
    w = cfg()
    r = run_oracle(w)
    for m, mp in enumerate(w.models[:6]):
        T = pb.t_eff(w.slo_us[m], w.margin_permille)
        totals = mp.lat_us.astype(np.int64).sum(axis=1)  # [C][B], whole model on one class
        for k in range(w.n_classes):
            pts = seg_points(r, w, m, 1, (k,))
            feas = [bi for bi in range(w.n_batches) if totals[k, bi] <= T]
            assert (len(pts) > 0) == (len(feas) > 0)
            if not feas:
                continue
            bidx = {int(b): i for i, b in enumerate(w.batches)}
            for p in pts:
                assert int(p["e2e_us"]) == totals[k, bidx[int(p["batch"])]]
            best = max(Fraction(int(w.batches[bi]), int(totals[k, bi])) for bi in feas)
            last = pts[-1]
            assert Fraction(int(last["batch"]), int(last["e2e_us"])) == best
            assert int(pts[0]["e2e_us"]) == min(totals[k, bi] for bi in feas)


# ---------------- P7: textbook min-max contiguous partition ----------------

def opt_minmax_partition(x, K):
    """Linear partition problem by dynamic programming (independent textbook routine)."""
    n = len(x)
    pre = [0]
    for v in x:
        pre.append(pre[-1] + int(v))
    INF = float("inf")
    dp = [[INF] * (n + 1) for _ in range(K + 1)]
    dp[0][0] = 0
    for k in range(1, K + 1):
        for j in range(1, n + 1):
            for i in range(k - 1, j):
                dp[k][j] = min(dp[k][j], max(dp[k - 1][i], pre[j] - pre[i]))
    return dp[K][n]


@pytest.mark.parametrize("seed", range(8))
def test_p7_linear_partition_special_case(oracle_built, seed):
    rng = np.random.default_rng(seed)
    M = int(rng.integers(3, 11))
    x = rng.integers(0, 50, size=M)
    x[0] += 1
    w = make_workload([x[None, :]], [[0] * M], 1000, [3], 10**6, margin=0, kmax=3)
    r = run_oracle(w)
    for K in (2, 3):
        pts = seg_points(r, w, 0, K, (0,) * K)
        assert len(pts) == 1  # S = 0: every candidate has E = total, so one frontier point
        p = pts[0]
        assert int(p["e2e_us"]) == int(x.sum())
        assert int(max(p["stage_us"][:K])) == opt_minmax_partition(list(x), K)
        # canonical: lexicographically smallest optimal cut tuple
        best = min(cuts for cuts in itertools.combinations(range(1, M), K - 1)
                   if max(int(x[a:b].sum()) for a, b in zip((0,) + cuts, cuts + (M,))) ==
                   opt_minmax_partition(list(x), K))
        assert tuple(int(c) for c in p["cut"][:K - 1]) == best


# ---------------- P8: literal O(n^2) Pareto definition ----------------

def compare_with_literal(w, r, use_np=False, vgpu=None):
    n_cand_total = 0
    for m in range(len(w.models)):
        segs, n_cand = pb.enumerate_candidates(w, m, vgpu=vgpu)
        n_cand_total += n_cand
        C, M = w.n_classes, w.models[m].n_layers
        for K in range(1, min(w.kmax, M) + 1):
            for cls in itertools.product(range(C), repeat=K):
                cands = segs.get((K, cls), [])
                lit = (pb.literal_frontier_np if use_np else pb.literal_frontier)(cands)
                got = seg_points(r, w, m, K, cls)
                assert len(got) == len(lit), (m, K, cls, len(got), len(lit))
                for g, e in zip(got, lit):
                    assert int(g["e2e_us"]) == e["E"]
                    assert int(g["batch"]) == e["b"]
                    assert (int(g["cut"][0]), int(g["cut"][1])) == e["cuts"]
                    assert [int(v) for v in g["stage_us"][:K]] == e["stages"]
                    assert list(g["cls"][:K]) == list(cls)
                    assert int(g["K"]) == K and int(g["model"]) == m
    assert r.n_candidates == n_cand_total


@pytest.mark.parametrize("seed", range(60))
def test_p8_literal_pareto_fuzz(oracle_built, seed):
    w = random_tiny(seed, n_models=1 + seed % 2)
    r = run_oracle(w, threads=1 + seed % 3)
    compare_with_literal(w, r)


def test_p8_literal_pareto_config1(oracle_built):
    w = config1()
    compare_with_literal(w, run_oracle(w))


@pytest.mark.slow
def test_p8_literal_pareto_config2(oracle_built):
    w = config2()
    compare_with_literal(w, run_oracle(w), use_np=True)


# ---------------- P10: virtual GPUs (App. A.2) ----------------
# A pseudo-class k on 1/v_k of a GPU: per-GPU stage throughput v_k b / C_d, plan
# throughput min over stages. Pinned by the literal definition with Fractions.

@pytest.mark.parametrize("seed", range(40))
def test_p10_vgpu_literal_pareto_fuzz(oracle_built, seed):
    w = random_tiny(seed, n_models=1 + seed % 2)
    rng = np.random.default_rng(seed)
    v = [int(x) for x in rng.integers(1, 5, size=w.n_classes)]
    compare_with_literal(w, run_oracle(w, threads=1 + seed % 2, vgpu=v), vgpu=v)


def test_p10_vgpu_uniform_scaling_is_neutral(oracle_built):
    """Scaling every v by the same factor scales every theta alike: same frontier."""
    w = config2()
    base = run_oracle(w)
    for v in (2, 3, 4):
        r = run_oracle(w, vgpu=[v] * w.n_classes)
        assert np.array_equal(r.points.view(np.uint8), base.points.view(np.uint8)), v


def test_p10_vgpu_hand_worked_bottleneck_moves(oracle_built):
    """M = 3 layers of 10, 20, 30 us on two classes with identical profiles, b = 1, no
    transfer cost, K = 2. Both cuts have E = 60: c = 1 gives C = (10, 50), c = 2 gives
    C = (30, 30), so one point per segment survives, the one with the larger theta.
    All v = 1: theta(c=1) = 1/50 < theta(c=2) = 1/30 -> c = 2 everywhere.
    v = (1, 2): segment (0, 1): c=1 runs its stages at 1/10 and 2/50 per GPU -> 1/25,
    c=2 at 1/30 and 2/30 -> 1/30, so c = 1 wins; segment (1, 0): c=1 -> min(2/10, 1/50)
    = 1/50, c=2 -> min(2/30, 1/30) = 1/30, so c = 2 stays."""
    from tests.fixtures import make_workload
    lat = np.array([[[10], [20], [30]], [[10], [20], [30]]], dtype=np.uint32)
    w = make_workload([lat], [[0, 0, 0]], 1000, [1], 10**6, margin=0, kmax=2)

    def k2_cut(r, cls):
        pts = [p for p in r.points if int(p["K"]) == 2 and tuple(int(c) for c in p["cls"][:2]) == cls]
        assert len(pts) == 1 and int(pts[0]["e2e_us"]) == 60
        return int(pts[0]["cut"][0])

    base = run_oracle(w)
    assert [k2_cut(base, c) for c in [(0, 0), (0, 1), (1, 0), (1, 1)]] == [2, 2, 2, 2]
    r = run_oracle(w, vgpu=[1, 2])
    assert [k2_cut(r, c) for c in [(0, 0), (0, 1), (1, 0), (1, 1)]] == [2, 1, 2, 2]
    compare_with_literal(w, r, vgpu=[1, 2])


# ---------------- invariants on the oracle ----------------

def frontier_set(r, w, m, K, cls):
    return [(int(p["e2e_us"]), int(p["batch"]), int(p["cut"][0]), int(p["cut"][1]))
            for p in seg_points(r, w, m, K, cls)]


def test_i3_slo_prefix_and_monotone_feasible(oracle_built):
    w = config2()
    slo_hi = 200000
    r_hi = run_oracle(w)
    feas_prev = -1
    for slo in (60000, 90000, 140000, 200000):
        r = run_oracle(w, slo_us=np.array([slo], dtype=np.uint32))
        T = pb.t_eff(slo, w.margin_permille)
        assert r.n_feasible >= feas_prev
        feas_prev = r.n_feasible
        for K in (1, 2, 3):
            for cls in itertools.product(range(3), repeat=K):
                lo = frontier_set(r, w, 0, K, cls)
                hi = [p for p in frontier_set(r_hi, w, 0, K, cls) if p[0] <= T]
                assert lo == hi
    assert slo_hi == 200000


def test_i4_raising_bandwidth(oracle_built):
    w = config2()
    r0 = run_oracle(w)
    w.bw = w.bw * 2
    r1 = run_oracle(w)
    assert r1.n_feasible >= r0.n_feasible


def test_i5_class_relabel_permutes_segments(oracle_built):
    w = config2()
    r0 = run_oracle(w)
    perm = [2, 0, 1]  # new class i = old class perm[i]
    w2 = make_workload([w.models[0].lat_us[perm]], [w.models[0].act_bytes], w.bw[np.ix_(perm, perm)],
                       w.batches, w.slo_us, w.margin_permille, 3)
    r1 = run_oracle(w2)
    inv = {old: new for new, old in enumerate(perm)}
    for K in (1, 2, 3):
        for cls in itertools.product(range(3), repeat=K):
            assert frontier_set(r0, w, 0, K, cls) == frontier_set(r1, w2, 0, K, tuple(inv[c] for c in cls))


def test_i6_i7_strict_staircase_and_direct_sums(oracle_built):
    w = config3()
    r = run_oracle(w)
    for s in range(len(r.seg_offsets) - 1):
        seg = r.points[int(r.seg_offsets[s]):int(r.seg_offsets[s + 1])]
        for a, b in zip(seg[:-1], seg[1:]):
            assert int(a["e2e_us"]) < int(b["e2e_us"])
            ta = Fraction(int(a["batch"]), max(int(x) for x in a["stage_us"]))
            tb = Fraction(int(b["batch"]), max(int(x) for x in b["stage_us"]))
            assert ta < tb
    bidx = {int(b): i for i, b in enumerate(w.batches)}
    for p in r.points[::7]:
        m, K = int(p["model"]), int(p["K"])
        mp = w.models[m]
        bounds = [0] + [int(c) for c in p["cut"][:K - 1]] + [mp.n_layers]
        bi = bidx[int(p["batch"])]
        st = [int(mp.lat_us[p["cls"][d], bounds[d]:bounds[d + 1], bi].astype(np.int64).sum()) for d in range(K)]
        assert st == [int(x) for x in p["stage_us"][:K]]
        y = sum(-(-8 * int(mp.act_bytes[bounds[d + 1] - 1]) * int(p["batch"]) //
                  int(w.bw[p["cls"][d], p["cls"][d + 1]])) for d in range(K - 1))
        assert int(p["e2e_us"]) == sum(st) + y <= pb.t_eff(w.slo_us[m], w.margin_permille)


def test_i8_duplicate_model_duplicates_segments(oracle_built):
    w = config3().subset([3, 3])
    r = run_oracle(w)
    n = (len(r.seg_offsets) - 1) // 2
    a = r.points[:int(r.seg_offsets[n])].copy()
    b = r.points[int(r.seg_offsets[n]):].copy()
    b["model"] = 0
    assert np.array_equal(a, b)


def test_thread_count_independence(oracle_built):
    w = config3()
    r1 = run_oracle(w, threads=1)
    r4 = run_oracle(w, threads=4)
    assert np.array_equal(r1.points, r4.points) and np.array_equal(r1.seg_offsets, r4.seg_offsets)
    assert (r1.n_candidates, r1.n_feasible) == (r4.n_candidates, r4.n_feasible)


def test_segment_filter_matches_full_run(oracle_built):
    w = config2()
    r = run_oracle(w)
    for K, cls in [(1, (2,)), (2, (0, 1)), (3, (1, 2, 0)), (3, (0, 0, 0))]:
        rs = run_oracle(w, only_K=K, only_cls=cls)
        got = rs.points
        exp = seg_points(r, w, 0, K, cls)
        assert np.array_equal(got, exp)
