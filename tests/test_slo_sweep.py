"""SLO sweeps from one enumeration (Fig. 12a).

ppipe_frontier_at derives the frontier at lower per-model latency targets by
truncating every segment of the last ppipe_pareto result (invariant I3). The bar
is the same as for the main path: bit-exact records and segment CSR against the
CPU oracle run directly at the lower SLO (and against a fresh GPU enumeration).
"""
from __future__ import annotations

import numpy as np
import pytest

import paper_2507_18748_b200 as pp
from oracle import run_oracle
from tests.helpers import assert_same_points
from workloads import config1, config2, config3, config5, random_tiny

pytestmark = pytest.mark.gpu


def _same(g, o, label):
    assert g.n_candidates == o.n_candidates, label
    assert_same_points(g.points, o.points, label)
    assert np.array_equal(g.seg_offsets, o.seg_offsets), label


@pytest.mark.parametrize("cfg", [config1, config2, config3])
def test_truncation_matches_oracle_at_lower_slo(oracle_built, cfg):
    w = cfg()
    ctx = pp.load_workload(w)
    try:
        base = (w.slo_us * 2).astype(np.uint32)  # enumerate once at twice the SLO
        pp.enumerate(ctx, w.kmax, base, w.margin_permille)
        pp.pareto(ctx)
        for scale, margin in [(2.0, w.margin_permille), (1.0, w.margin_permille), (0.5, w.margin_permille),
                              (1.0, 600), (2.0, 999), (0.05, 0)]:
            slo = (w.slo_us * scale).astype(np.uint32)
            T_new = slo.astype(np.int64) * (1000 - margin) // 1000
            T_base = base.astype(np.int64) * (1000 - w.margin_permille) // 1000
            if (T_new > T_base).any():
                continue
            g = pp.frontier_at(ctx, slo, margin)
            o = run_oracle(w, slo_us=slo, margin_permille=margin)
            _same(g, o, f"{w.name} slo x{scale} margin {margin}")
    finally:
        pp.free(ctx)


@pytest.mark.parametrize("seed", range(16))
def test_truncation_random_per_model_targets(oracle_built, seed):
    w = random_tiny(seed, max_layers=10, n_models=1 + seed % 4)
    rng = np.random.default_rng(seed)
    ctx = pp.load_workload(w)
    try:
        pp.enumerate(ctx, w.kmax, w.slo_us, w.margin_permille)
        pp.pareto(ctx)
        for _ in range(3):
            slo = (w.slo_us * rng.uniform(0.0, 1.0, size=len(w.slo_us))).astype(np.uint32)
            g = pp.frontier_at(ctx, slo, w.margin_permille)
            _same(g, run_oracle(w, slo_us=slo), f"tiny {seed}")
    finally:
        pp.free(ctx)


def test_truncation_equals_fresh_enumeration_config5_slice():
    w = config5(n_models=24)
    ctx = pp.load_workload(w)
    try:
        pp.enumerate(ctx, 3, w.slo_us, w.margin_permille)
        pp.pareto(ctx)
        fronts = {}
        for scale in (0.9, 0.6, 0.3):
            slo = (w.slo_us * scale).astype(np.uint32)
            fronts[scale] = pp.frontier_at(ctx, slo, w.margin_permille)
        for scale, g in fronts.items():  # re-enumerate from scratch on a second context
            c2 = pp.load_workload(w)
            try:
                pp.enumerate(c2, 3, (w.slo_us * scale).astype(np.uint32), w.margin_permille)
                f = pp.pareto(c2)
            finally:
                pp.free(c2)
            assert f.n_points == g.n_points, scale
            assert np.array_equal(f.points.view(np.uint8), g.points.view(np.uint8)), scale
            assert np.array_equal(f.seg_offsets, g.seg_offsets), scale
    finally:
        pp.free(ctx)


def test_truncation_errors():
    w = config1()
    ctx = pp.load_workload(w)
    try:
        with pytest.raises(pp.PPipeError) as e:
            pp.frontier_at(ctx, w.slo_us, w.margin_permille)
        assert e.value.code == -6  # ESTATE: no pareto yet
        pp.enumerate(ctx, w.kmax, w.slo_us, w.margin_permille)
        with pytest.raises(pp.PPipeError) as e:
            pp.frontier_at(ctx, w.slo_us, w.margin_permille)
        assert e.value.code == -6  # enumerate without pareto
        pp.pareto(ctx)
        with pytest.raises(pp.PPipeError) as e:
            pp.frontier_at(ctx, w.slo_us * 2, w.margin_permille)
        assert e.value.code == -1  # a sweep can only lower the target
        g = pp.frontier_at(ctx, w.slo_us, w.margin_permille)  # same target: the pareto result itself
        assert g.n_points == pp.pareto(ctx).n_points
    finally:
        pp.free(ctx)
