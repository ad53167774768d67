"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Integer results, so the bar is bit-exact equality of every frontier record,
the segment CSR, and the candidate / feasible counts (north_star).
"""
from __future__ import annotations

import numpy as np
import pytest

import paper_2507_18748_b200 as pp
from oracle import run_oracle
from tests.fixtures import make_workload
from tests.helpers import (assert_same_points, assert_same_result, reduce_union, seg_index_of, segment_points)
from workloads import config1, config2, config3, config4, config5, random_tiny

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg", [config1, config2, config3])
def test_parity_small_configs(oracle_built, cfg):
    w = cfg()
    assert_same_result(pp.run(w), run_oracle(w), w.name)


def test_parity_config4_full(oracle_built):
    w = config4()
    g = pp.run(w)
    o = run_oracle(w)
    assert g.n_candidates == 994806720
    assert_same_result(g, o, "config 4")


@pytest.mark.parametrize("seed", range(120))
def test_parity_random_tiny(oracle_built, seed):
    w = random_tiny(seed, max_layers=10, n_models=1 + seed % 3)
    assert_same_result(pp.run(w), run_oracle(w), f"tiny {seed}")


@pytest.mark.parametrize("seed", range(12))
def test_parity_random_medium(oracle_built, seed):
    # several 32*kJ1 first-cut tiles and ragged tails; C up to 8 (largest template)
    rng = np.random.default_rng(1000 + seed)
    C = [1, 2, 3, 5, 8, 4, 6, 7][seed % 8]
    M = int(rng.integers(130, 420))
    B = int(rng.integers(1, 6))
    batches = np.sort(rng.choice(np.arange(1, 40), size=B, replace=False))
    lat = (rng.lognormal(4, 1, size=(C, M, B)) * (1 + np.arange(B))[None, None, :]).astype(np.uint32)
    lat[rng.random(lat.shape) < 0.05] = 0
    S = (rng.lognormal(11, 1.5, size=M)).astype(np.uint64)
    bw = rng.choice([2000, 6400, 10000], size=(C, C))
    tot = lat.astype(np.int64).sum(axis=1).min()
    w = make_workload([lat], [S], bw, batches, int(tot * 2.2), margin=400, kmax=3)
    assert_same_result(pp.run(w), run_oracle(w), f"medium {seed}")


def test_edge_shapes(oracle_built):
    cases = [
        make_workload([[[5]]], [[7]], 1, [1], 100, kmax=3),                       # M = 1
        make_workload([[[5, 0]], [[0, 5]]], [[100, 0], [0, 0]], 3, [1], 100, kmax=3),  # M = 2, Cmax = 0
        make_workload([np.zeros((2, 3, 1), np.uint32)], [[1, 2, 3]], 1, [2], 1000, kmax=3),  # all-zero latency
        make_workload([np.ones((1, 5, 1), np.uint32) * 9], [[0] * 5], 7, [1], 10, kmax=3),  # nothing feasible
        make_workload([np.ones((2, 6, 2), np.uint32)], [[10**9] * 6], 1, [1, 2], 10**7, kmax=3),  # Y clamps
    ]
    for i, w in enumerate(cases):
        assert_same_result(pp.run(w), run_oracle(w), f"edge {i}")


def test_many_batches_pack_tiles(oracle_built):
    # B > 64 exercises several batch tiles in the pack kernel
    rng = np.random.default_rng(7)
    B = 150
    lat = rng.integers(0, 40, size=(2, 12, B)).astype(np.uint32)
    w = make_workload([lat], [rng.integers(0, 5000, size=12)], 4000, np.arange(1, B + 1), 600, kmax=3)
    assert_same_result(pp.run(w), run_oracle(w), "B=150")


def test_kmax_variants(oracle_built):
    for kmax in (1, 2, 3):
        w = config2()
        w.kmax = kmax
        assert_same_result(pp.run(w), run_oracle(w), f"config 2 kmax {kmax}")


def test_slo_and_margin_sweep_reuse_context(oracle_built):
    w = config3()
    ctx = pp.load_workload(w)
    try:
        for scale, margin in [(1.0, 400), (0.5, 400), (2.0, 200), (1.0, 0), (0.1, 999)]:
            slo = (w.slo_us * scale).astype(np.uint32)
            pp.enumerate(ctx, 3, slo, margin)
            g = pp.pareto(ctx)
            o = run_oracle(w, slo_us=slo, margin_permille=margin)
            assert_same_result(g, o, f"slo x{scale} margin {margin}")
    finally:
        pp.free(ctx)


def test_survivor_buffer_regrowth(oracle_built, monkeypatch):
    """A survivor buffer that is too small is grown and the enumeration re-run;
    the result must not change (PPIPE_SURVIVOR_CAP sets the initial capacity)."""
    monkeypatch.setenv("PPIPE_SURVIVOR_CAP", "16")
    w = config3()
    g = pp.run(w)
    assert g.n_survivors > 16
    assert_same_result(g, run_oracle(w), "regrowth")


@pytest.mark.parametrize("cap", ["1", "7"])
def test_hot_unit_buffer_regrowth(oracle_built, monkeypatch, cap):
    """A hot-unit buffer (pass-1 tables handed to pass 2) that is too small is grown and
    the enumeration re-run; the result must not change (PPIPE_HOT_CAP sets the initial
    capacity; the overflowing units still push their staircases into the global fold)."""
    monkeypatch.setenv("PPIPE_HOT_CAP", cap)
    for w in (config3(), config5(model_ids=[4, 17])):
        assert_same_result(pp.run(w), run_oracle(w), f"hot-unit regrowth from {cap}, {w.name}")


def test_determinism(oracle_built):
    w = config3()
    a, b = pp.run(w), pp.run(w)
    assert_same_points(a.points, b.points, "rerun")


@pytest.mark.parametrize("world", [2, 3, 5])
def test_shard_mode_local_frontiers_and_union(oracle_built, world):
    """Each rank's local frontier equals the oracle over that rank's rows; the
    union of local frontiers reduces to the single-GPU frontier."""
    w = config3()
    full = pp.run(w)
    parts = []
    Ms = [m.n_layers for m in w.models]
    for r in range(world):
        rows = pp.partition_rows(Ms, w.n_classes, w.n_batches, 3, r, world)
        ctx = pp.load_workload(w, rank=r, world=world)
        try:
            pp.enumerate(ctx, w.kmax, w.slo_us, w.margin_permille)
            g = pp.pareto(ctx)
        finally:
            pp.free(ctx)
        parts.append(g.points)
        for m in range(len(w.models)):
            lo, hi = int(rows[m, 0]), int(rows[m, 1])
            if hi <= lo:
                continue
            o = run_oracle(w, model_lo=m, model_hi=m + 1, row_lo=lo, row_hi=hi)
            mine = g.points[g.points["model"] == m]
            assert_same_points(mine, o.points, f"rank {r} model {m} rows [{lo},{hi})")
    union = np.concatenate(parts)
    assert_same_points(reduce_union(union), full.points, f"union of {world} shards")


def test_large_model_global_B_path(oracle_built):
    """M > 8192 takes the kernel variant that reads B(c2) from global memory.
    Checked on a shard (few first-cut rows) against the oracle's row filter."""
    rng = np.random.default_rng(11)
    M = 8300
    lat = rng.integers(0, 3, size=(2, M, 1)).astype(np.uint32)
    S = rng.integers(0, 2000, size=M)
    w = make_workload([lat], [S], 8000, [1], int(lat.sum(axis=1).min() * 1.5), kmax=3)
    world, rank = 4000, 3997
    rows = pp.partition_rows([M], 2, 1, 3, rank, world)
    lo, hi = int(rows[0, 0]), int(rows[0, 1])
    assert hi > lo
    ctx = pp.load_workload(w, rank=rank, world=world)
    try:
        pp.enumerate(ctx, 3, w.slo_us, w.margin_permille)
        g = pp.pareto(ctx)
    finally:
        pp.free(ctx)
    o = run_oracle(w, row_lo=lo, row_hi=hi)
    assert g.n_candidates == o.n_candidates and g.n_feasible == o.n_feasible
    assert_same_points(g.points, o.points, "M=8300 shard")


def test_config5_sampled_models(oracle_built):
    """Two whole config-5 models (smallest M) against the oracle."""
    ids = [4, 17]
    w = config5(model_ids=ids)
    assert_same_result(pp.run(w), run_oracle(w), "config 5 models 4, 17")


def test_config5_full_size_sampled_segments(oracle_built):
    """The full 1,000-model config-5 run (the launch bench.py times), checked
    on sampled segments the oracle computes one by one, plus invariants."""
    w = config5()
    g = pp.run(w)
    C = w.n_classes
    total = sum(sum(C ** k for k in range(1, 4)) for _ in w.models)
    assert g.n_segments == total and len(g.seg_offsets) == total + 1
    rng = np.random.default_rng(5)
    small = sorted(range(len(w.models)), key=lambda m: w.models[m].n_layers)[:40]
    for m in rng.choice(small, size=3, replace=False):
        m = int(m)
        for K, cls in [(3, tuple(int(x) for x in rng.integers(0, C, 3))), (2, (4, 1)), (1, (4,))]:
            o = run_oracle(w, model_lo=m, model_hi=m + 1, only_K=K, only_cls=cls)
            s = seg_index_of(w, m, K, cls)
            got = segment_points(g.points, g.seg_offsets, s)
            assert_same_points(got, o.points, f"config 5 model {m} K={K} cls={cls}")
    check_invariants(w, g)


def check_invariants(w, g, every=97):
    pts = g.points
    # I6: along each segment E and theta strictly increase
    for s in range(0, int(g.n_segments), every):
        seg = segment_points(pts, g.seg_offsets, s)
        if len(seg) < 2:
            continue
        E = seg["e2e_us"].astype(np.int64)
        cm = seg["stage_us"].max(axis=1).astype(np.int64)
        b = seg["batch"].astype(np.int64)
        assert (np.diff(E) > 0).all()
        assert (b[1:] * cm[:-1] > b[:-1] * cm[1:]).all()
    # I7: stored stages equal direct sums, E - sum(C) equals the recomputed transfers, E <= T_eff
    bidx = {int(x): i for i, x in enumerate(w.batches)}
    for p in pts[::max(1, len(pts) // 500)]:
        m, K = int(p["model"]), int(p["K"])
        mp = w.models[m]
        bounds = [0] + [int(c) for c in p["cut"][:K - 1]] + [mp.n_layers]
        bi = bidx[int(p["batch"])]
        st = [int(mp.lat_us[p["cls"][d], bounds[d]:bounds[d + 1], bi].astype(np.int64).sum()) for d in range(K)]
        assert st == [int(x) for x in p["stage_us"][:K]]
        y = sum(-(-8 * int(mp.act_bytes[bounds[d + 1] - 1]) * int(p["batch"]) //
                  int(w.bw[p["cls"][d], p["cls"][d + 1]])) for d in range(K - 1))
        assert int(p["e2e_us"]) == sum(st) + y
        assert int(p["e2e_us"]) <= int(w.slo_us[m]) * (1000 - w.margin_permille) // 1000


def test_invariants_config4(oracle_built):
    w = config4()
    check_invariants(w, pp.run(w), every=1)


def test_errors_on_device():
    w = config1()
    ctx = pp.load_workload(w)
    try:
        with pytest.raises(pp.PPipeError) as e:
            pp.pareto(ctx)
        assert e.value.code == -6  # ESTATE
        with pytest.raises(pp.PPipeError) as e:
            pp.enumerate(ctx, 4, w.slo_us, 400)
        assert e.value.code == -1
        with pytest.raises(pp.PPipeError) as e:
            pp.enumerate(ctx, 3, w.slo_us, 1000)
        assert e.value.code == -1
        with pytest.raises(pp.PPipeError) as e:
            pp.enumerate(ctx, 3, np.array([1 << 30], np.uint32), 0)
        assert e.value.code == -2
    finally:
        pp.free(ctx)


def test_update_profiles_validates_on_device(oracle_built):
    """ppipe_update_profiles checks the int32 envelope on the GPU after the copy; the
    error names the same item as the host check of ppipe_load_profiles, the context
    refuses to enumerate until a good update, and then computes the right result."""
    w = config3()
    lat = [m.lat_us.copy() for m in w.models]
    S = [m.act_bytes.copy() for m in w.models]
    ctx = pp.load_workload(w)
    try:
        bad = [x.copy() for x in lat]
        bad[5][2, :, 7] = (1 << 28) // bad[5].shape[1] + 1  # class 2, batch index 7 of model 5
        bad[9][1, :, 3] = (1 << 28) // bad[9].shape[1] + 1
        with pytest.raises(pp.PPipeError) as e:
            pp.update_profiles(ctx, bad, S)
        assert e.value.code == -2
        assert f"model 5 class 2 batch {int(w.batches[7])}: whole-model latency" in str(e.value)
        with pytest.raises(pp.PPipeError) as e2:
            ppl = pp.load_profiles(bad, S, w.n_classes, w.batches, w.bw)  # host check, same message
            pp.free(ppl)
        assert str(e2.value).split(": ", 1)[-1] == str(e.value).split(": ", 1)[-1]
        with pytest.raises(pp.PPipeError) as e3:
            pp.enumerate(ctx, w.kmax, w.slo_us, w.margin_permille)
        assert e3.value.code == -6
        badS = [x.copy() for x in S]
        badS[4][3] = np.uint64(1 << 62)
        with pytest.raises(pp.PPipeError) as e4:
            pp.update_profiles(ctx, lat, badS)
        assert "model 4 layer 3: act_bytes" in str(e4.value)
        pp.update_profiles(ctx, lat, S)
        pp.enumerate(ctx, w.kmax, w.slo_us, w.margin_permille)
        assert_same_result(pp.pareto(ctx), run_oracle(w), "after a good update")
    finally:
        pp.free(ctx)


@pytest.mark.parametrize("split", ["1", "3"])
def test_frontier_pass_large_segment_paths(oracle_built, monkeypatch, split):
    """Segments above the CTA path's shared-memory capacity (kFpCap = 4096 survivors)
    are split by E ranges into sub-segments; PPIPE_FP_SPLIT fixes the number of
    sub-segments so that the last-resort global-memory merge sort (split = 1: every
    large segment whole) and uneven splits run. Result: bit-exact vs the oracle."""
    monkeypatch.setenv("PPIPE_FP_SPLIT", split)
    w = config4()
    g = pp.run(w)
    assert_same_result(g, run_oracle(w), f"config 4, PPIPE_FP_SPLIT={split}")
