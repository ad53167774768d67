"""GPU parity of F2, the MILP-lossless frontier (ppipe_pareto_f2),
against the oracle's literal all-pairs F2 reduction (oracle/ppipe_oracle.c f2_beats,
pinned by tests/test_f2_pins.py). Integer results: records, CSR and counts must be
byte-identical.
"""
from __future__ import annotations

import itertools

import numpy as np
import pytest

import paper_2507_18748_b200 as pp
from oracle import run_oracle
from tests.fixtures import make_workload
from tests.helpers import assert_same_points, assert_same_result, seg_index_of, segment_points
from workloads import config1, config2, config3, config4, config5, random_tiny

pytestmark = pytest.mark.gpu


def f2(w, **kw):
    return pp.run(w, frontier=2, **kw)


@pytest.mark.parametrize("cfg", [config1, config2, config3])
def test_f2_parity_small_configs(oracle_built, cfg):
    w = cfg()
    assert_same_result(f2(w), run_oracle(w, frontier=2), w.name)


@pytest.mark.parametrize("seed", range(100))
def test_f2_parity_random_tiny(oracle_built, seed):
    w = random_tiny(seed, max_layers=10, n_models=1 + seed % 3)
    assert_same_result(f2(w), run_oracle(w, frontier=2), f"tiny {seed}")


@pytest.mark.parametrize("seed", range(10))
def test_f2_parity_random_medium(oracle_built, seed):
    # several warps of c_1 rows and ragged 32-wide c_2 groups; zero-latency layers make ties
    rng = np.random.default_rng(2000 + seed)
    C = [1, 2, 3, 2, 4][seed % 5]
    M = int(rng.integers(40, 140 if C <= 2 else 70))
    B = int(rng.integers(1, 6))
    batches = np.sort(rng.choice(np.arange(1, 40), size=B, replace=False))
    lat = (rng.lognormal(4, 1, size=(C, M, B)) * (1 + np.arange(B))[None, None, :]).astype(np.uint32)
    lat[rng.random(lat.shape) < 0.05] = 0
    S = (rng.lognormal(11, 1.5, size=M)).astype(np.uint64)
    bw = rng.choice([2000, 6400, 10000], size=(C, C))
    tot = lat.astype(np.int64).sum(axis=1).min()
    w = make_workload([lat], [S], bw, batches, int(tot * 2.2), margin=400, kmax=3)
    assert_same_result(f2(w), run_oracle(w, frontier=2), f"medium {seed}")


def test_f2_edge_shapes(oracle_built):
    cases = [
        make_workload([[[5]]], [[7]], 1, [1], 100, kmax=3),                       # M = 1
        make_workload([[[5, 0]], [[0, 5]]], [[100, 0], [0, 0]], 3, [1], 100, kmax=3),  # M = 2, a stage of 0 us
        make_workload([np.zeros((2, 3, 2), np.uint32)], [[1, 2, 3]], 1, [2, 4], 1000, kmax=3),  # all-zero: +inf ties
        make_workload([np.ones((1, 5, 1), np.uint32) * 9], [[0] * 5], 7, [1], 10, kmax=3),  # nothing feasible
        make_workload([np.ones((2, 6, 2), np.uint32)], [[10**9] * 6], 1, [1, 2], 10**7, kmax=3),  # Y clamps
        make_workload([np.array([[[2, 4], [4, 8], [6, 12]]], np.uint32)], [[0, 0, 0]], 1, [1, 2], 10**4,
                      kmax=3),  # lat(b=2) = 2 lat(b=1): every vector tied across batches
    ]
    for i, w in enumerate(cases):
        assert_same_result(f2(w), run_oracle(w, frontier=2), f"edge {i}")


def test_f2_kmax_variants_and_vgpu_neutral(oracle_built):
    for kmax in (1, 2, 3):
        w = config2()
        w.kmax = kmax
        assert_same_result(f2(w), run_oracle(w, frontier=2), f"kmax {kmax}")
    w = config3()
    v = [1, 2, 3, 4][:w.n_classes]
    assert_same_result(f2(w, vgpu=v), run_oracle(w, frontier=2), "vgpu")


def test_f2_many_batches(oracle_built):
    rng = np.random.default_rng(8)
    B = 70
    lat = rng.integers(0, 40, size=(2, 9, B)).astype(np.uint32)
    w = make_workload([lat], [rng.integers(0, 5000, size=9)], 4000, np.arange(1, B + 1), 400, kmax=3)
    assert_same_result(f2(w), run_oracle(w, frontier=2), "B=70")


def test_f2_survivor_regrowth_and_g_chunks(oracle_built, monkeypatch):
    """A tiny G budget forces one K = 3 segment per chunk; results must not change."""
    monkeypatch.setenv("PPIPE_F2_G_BYTES", "1")
    w = config3()
    assert_same_result(f2(w), run_oracle(w, frontier=2), "G chunks")


def test_f2_reuses_context_with_the_staircase(oracle_built):
    """ppipe_pareto_f2 and ppipe_enumerate/ppipe_pareto on one context, in both orders."""
    w = config2()
    ctx = pp.load_workload(w)
    try:
        a = pp.pareto_f2(ctx, w.kmax, w.slo_us, w.margin_permille)
        pp.enumerate(ctx, w.kmax, w.slo_us, w.margin_permille)
        b = pp.pareto(ctx)
        c = pp.pareto_f2(ctx, w.kmax, w.slo_us // 2, w.margin_permille)
    finally:
        pp.free(ctx)
    assert_same_result(a, run_oracle(w, frontier=2), "f2 first")
    assert_same_result(b, run_oracle(w), "staircase after f2")
    assert_same_result(c, run_oracle(w, frontier=2, slo_us=w.slo_us // 2), "f2 at half the SLO")


@pytest.mark.parametrize("world", [2, 3])
def test_f2_shard_mode_owns_whole_models(oracle_built, world):
    """Shard mode: each rank returns the F2 points of the models whose K = 1 row it holds;
    their concatenation in rank order is the single-GPU result."""
    w = config3()
    full = f2(w)
    parts = [f2(w, rank=r, world=world).points for r in range(world)]
    assert_same_points(np.concatenate(parts), full.points, f"{world} shards")


def test_f2_config4_sampled_segments(oracle_built):
    """config 4 (the F2 bench workload, 994,806,720 candidates): every K <= 2 segment and
    eight K = 3 segments against the oracle, plus the counts."""
    w = config4()
    g = f2(w)
    assert g.n_candidates == 994806720
    o2 = run_oracle(w, only_K=0, kmax=2, frontier=2)
    assert g.n_feasible == run_oracle(w).n_feasible
    C = w.n_classes
    for K in (1, 2):
        for cls in itertools.product(range(C), repeat=K):
            s = seg_index_of(w, 0, K, cls)
            got = segment_points(g.points, g.seg_offsets, s)
            exp = segment_points(o2.points, o2.seg_offsets, sum(C ** k for k in range(1, K)) +
                                 int(np.ravel_multi_index(cls, (C,) * K)))
            assert_same_points(got, exp, f"config 4 K={K} cls={cls}")
    rng = np.random.default_rng(4)
    for _ in range(8):
        cls = tuple(int(x) for x in rng.integers(0, C, 3))
        o = run_oracle(w, only_K=3, only_cls=cls, frontier=2)
        got = segment_points(g.points, g.seg_offsets, seg_index_of(w, 0, 3, cls))
        assert_same_points(got, o.points, f"config 4 K=3 cls={cls}")


def test_f2_config5_sampled_model(oracle_built):
    """A whole deep config-5 model (M > 514 -> 4 G columns per thread) on sampled segments."""
    w = config5(model_ids=[0, 1, 2, 3])
    g = f2(w)
    m = max(range(4), key=lambda i: w.models[i].n_layers)
    assert w.models[m].n_layers > 514
    rng = np.random.default_rng(6)
    C = w.n_classes
    for K, cls in [(3, tuple(int(x) for x in rng.integers(0, C, 3))), (3, (0, 4, 1)), (2, (4, 1)), (1, (2,))]:
        o = run_oracle(w, model_lo=m, model_hi=m + 1, only_K=K, only_cls=cls, frontier=2)
        got = segment_points(g.points, g.seg_offsets, seg_index_of(w, m, K, cls))
        assert_same_points(got, o.points, f"config 5 model {m} K={K} cls={cls}")


def test_f2_errors():
    w = config1()
    ctx = pp.load_workload(w)
    try:
        with pytest.raises(pp.PPipeError):
            pp.pareto_f2(ctx, 4, w.slo_us, w.margin_permille)
        with pytest.raises(pp.PPipeError):
            pp.pareto_f2(ctx, 3, w.slo_us, 1000)
        pp.update_profiles_async(ctx, [m.lat_us for m in w.models], [m.act_bytes for m in w.models])
        with pytest.raises(pp.PPipeError) as e:
            pp.pareto_f2(ctx, 3, w.slo_us, w.margin_permille)
        assert "update_profiles_async" in str(e.value)
    finally:
        pp.free(ctx)


def test_f2_config4_whole_vs_oracle_golden():
    """F2 on the whole of config 4 (994.8M candidates, 2.2M F2 points) against the
    oracle's literal all-pairs F2, stored as hashes by scripts/golden_f2_config4.py
    (oracle only; 332 s on 8 host threads)."""
    import hashlib
    import json
    import os
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "f2_config4_oracle.json")
    gold = json.load(open(path))
    w = config4()
    g = pp.run(w, frontier=2)
    assert g.n_candidates == gold["n_cand"] and g.n_feasible == gold["n_feas"]
    assert g.n_points == gold["n_pts"]
    assert hashlib.sha256(np.ascontiguousarray(g.points).tobytes()).hexdigest() == gold["sha_pts"]
    seg = np.diff(g.seg_offsets.astype(np.uint64)).astype("<u8")
    assert hashlib.sha256(seg.tobytes()).hexdigest() == gold["sha_seg"]
