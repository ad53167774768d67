"""Virtual-GPU pseudo-classes (App. A.2).

A class on 1/v of a GPU delivers v * b / C per physical GPU, and a plan's throughput
is the minimum over its stages. Same bar as the main path: bit-exact records, CSR
and counts against the oracle run with the same v's.
"""
from __future__ import annotations

import numpy as np
import pytest

import paper_2507_18748_b200 as pp
from oracle import run_oracle
from tests.helpers import assert_same_result
from workloads import config1, config2, config3, config5, random_tiny

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg,v", [(config1, [1, 2]), (config2, [2, 1, 4]), (config3, [1, 2, 3, 4]),
                                   (config3, [4, 4, 2, 2])])
def test_vgpu_small_configs(oracle_built, cfg, v):
    w = cfg()
    assert_same_result(pp.run(w, vgpu=v), run_oracle(w, vgpu=v), f"{w.name} v={v}")


@pytest.mark.parametrize("seed", range(40))
def test_vgpu_random_tiny(oracle_built, seed):
    w = random_tiny(seed, max_layers=10, n_models=1 + seed % 3)
    v = [int(x) for x in np.random.default_rng(seed).integers(1, 5, size=w.n_classes)]
    assert_same_result(pp.run(w, vgpu=v), run_oracle(w, vgpu=v), f"tiny {seed} v={v}")


def test_vgpu_config5_models(oracle_built):
    """Two whole deep models (M ~ 600): the pass-2 tightening with weighted stages."""
    w = config5(n_models=2)
    v = [1, 2, 3, 4, 2]
    assert_same_result(pp.run(w, vgpu=v), run_oracle(w, vgpu=v), "config 5 x2")


def test_vgpu_default_and_reset(oracle_built):
    w = config2()
    base = pp.run(w)
    ctx = pp.load_workload(w)
    try:
        pp.set_vgpu(ctx, [2, 2, 2])  # uniform: same theta order, same frontier
        pp.enumerate(ctx, w.kmax, w.slo_us, w.margin_permille)
        g = pp.pareto(ctx)
        assert np.array_equal(g.points.view(np.uint8), base.points.view(np.uint8))
        pp.set_vgpu(ctx, [1, 4, 1])
        with pytest.raises(pp.PPipeError):
            pp.pareto(ctx)  # results invalidated
        pp.set_vgpu(ctx, None)
        pp.enumerate(ctx, w.kmax, w.slo_us, w.margin_permille)
        assert np.array_equal(pp.pareto(ctx).points.view(np.uint8), base.points.view(np.uint8))
        with pytest.raises(pp.PPipeError) as e:
            pp.set_vgpu(ctx, [1, 5, 1])
        assert e.value.code == -1
    finally:
        pp.free(ctx)
