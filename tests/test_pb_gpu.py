"""GPU parity of per-stage batch sizes (ppipe_pareto_pb)
against the oracle's brute force (oracle_run_pb, pinned by tests/test_pb_pins.py).
Integer results: records, CSR and counts must be byte-identical.
"""
from __future__ import annotations

import numpy as np
import pytest

import paper_2507_18748_b200 as pp
from oracle import run_oracle_pb
from tests.fixtures import make_workload
from tests.helpers import assert_same_result
from workloads import config1, config2, config3, random_tiny

pytestmark = pytest.mark.gpu


def pbrun(w, **kw):
    return pp.run(w, frontier=3, **kw)


@pytest.mark.parametrize("cfg", [config1, config2, config3])
def test_pb_parity_configs(oracle_built, cfg):
    w = cfg()
    assert_same_result(pbrun(w), run_oracle_pb(w), w.name)


@pytest.mark.parametrize("seed", range(80))
def test_pb_parity_random_tiny(oracle_built, seed):
    w = random_tiny(600 + seed, max_layers=9, max_batches=4, n_models=1 + seed % 3)
    assert_same_result(pbrun(w), run_oracle_pb(w), f"tiny {seed}")


@pytest.mark.parametrize("seed", range(6))
def test_pb_parity_random_medium(oracle_built, seed):
    # many first cuts and batches: units of up to (M - 2) * B^2 candidates, ragged tails
    rng = np.random.default_rng(3000 + seed)
    C = [1, 2, 3][seed % 3]
    M = int(rng.integers(12, 40))
    B = int(rng.integers(2, 12))
    batches = np.sort(rng.choice(np.arange(1, 65), size=B, replace=False))
    lat = (rng.lognormal(4, 1, size=(C, M, B)) * (1 + 0.3 * np.arange(B))[None, None, :]).astype(np.uint32)
    lat[rng.random(lat.shape) < 0.05] = 0
    S = (rng.lognormal(11, 1.5, size=M)).astype(np.uint64)
    bw = rng.choice([2000, 6400, 10000], size=(C, C))
    tot = lat.astype(np.int64).sum(axis=1).min()
    w = make_workload([lat], [S], bw, batches, int(tot * 2.5), margin=400, kmax=3)
    assert_same_result(pbrun(w), run_oracle_pb(w), f"medium {seed}")


def test_pb_edge_shapes(oracle_built):
    cases = [
        make_workload([[[5]]], [[7]], 1, [1], 100, kmax=3),
        make_workload([[[5, 0]], [[0, 5]]], [[100, 0], [0, 0]], 3, [1], 100, kmax=3),
        make_workload([np.zeros((2, 3, 2), np.uint32)], [[1, 2, 3]], 1, [2, 4], 1000, kmax=3),
        make_workload([np.ones((1, 5, 1), np.uint32) * 9], [[0] * 5], 7, [1], 10, kmax=3),
        make_workload([np.ones((2, 6, 2), np.uint32)], [[10**9] * 6], 1, [1, 2], 10**7, kmax=3),
        make_workload([np.array([[[40, 64], [5, 20]]], np.uint32)], [[0, 0]], 1000, [1, 4], 1000, kmax=2),
    ]
    for i, w in enumerate(cases):
        assert_same_result(pbrun(w), run_oracle_pb(w), f"edge {i}")


def test_pb_kmax_and_shards(oracle_built):
    for kmax in (1, 2, 3):
        w = config3()
        w.kmax = kmax
        assert_same_result(pbrun(w), run_oracle_pb(w), f"kmax {kmax}")
    w = config3()
    full = pbrun(w)
    parts = [pbrun(w, rank=r, world=3).points for r in range(3)]
    assert np.array_equal(np.concatenate(parts).view(np.uint8), full.points.view(np.uint8))


def test_pb_errors():
    w = config1()
    ctx = pp.load_workload(w)
    try:
        with pytest.raises(pp.PPipeError):
            pp.pareto_pb(ctx, 0, w.slo_us, w.margin_permille)
    finally:
        pp.free(ctx)
    many = make_workload([np.ones((1, 3, 256), np.uint32)], [[0, 0, 0]], 1, np.arange(1, 257), 10**6, kmax=2)
    ctx = pp.load_workload(many)
    try:
        with pytest.raises(pp.PPipeError) as e:
            pp.pareto_pb(ctx, 2, many.slo_us, 0)
        assert "255" in str(e.value)
    finally:
        pp.free(ctx)
