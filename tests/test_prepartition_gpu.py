"""GPU pre-partitioning (ppipe_prepartition) against the CPU oracle, bit-exact.

PAPER.md:1005-1010 (§5.2): greedy blocks of approximately equal runtime on one GPU
type; SURVEY.md §8(f) NEXT-3. Bounds, per-(class, batch) block latencies and block
output bytes must equal oracle_prepartition's exactly.
"""
from __future__ import annotations

import numpy as np
import pytest

import paper_2507_18748_b200 as pp
from oracle import prepartition_oracle
from workloads import config3, config5

pytestmark = pytest.mark.gpu


def _check(lat_list, S_list, N, rc, rb, label):
    bounds, blat, bS = pp.prepartition(lat_list, S_list, N, rc, rb)
    for m, (lat, S) in enumerate(zip(lat_list, S_list)):
        ob, olat, oS = prepartition_oracle(lat, S, N, rc, rb)
        assert np.array_equal(bounds[m], ob), (label, m, bounds[m], ob)
        assert np.array_equal(blat[m].astype(np.uint64), olat), (label, m)
        assert np.array_equal(bS[m], oS), (label, m)
    return bounds, blat, bS


@pytest.mark.parametrize("N", [1, 5, 10, 20])
def test_config3_layer_models(oracle_built, N):
    w = config3(n_blocks=None)
    _check([m.lat_us for m in w.models], [m.act_bytes for m in w.models], N, 1, 0, f"3L N={N}")


def test_config3_blocks_feed_the_planner(oracle_built):
    """The block profiles are planner input: N=10 blocks of the 3L models on the
    L4-like class at batch 1 reproduce config 3's models (its generator applies the
    same rule), and enumerating them gives config 3's frontier."""
    w3, wl = config3(), config3(n_blocks=None)
    bounds, blat, bS = pp.prepartition([m.lat_us for m in wl.models], [m.act_bytes for m in wl.models], 10, 1, 0)
    for m in range(len(w3.models)):
        assert np.array_equal(blat[m], w3.models[m].lat_us), m
        assert np.array_equal(bS[m], w3.models[m].act_bytes), m
    g1 = pp.run(w3)
    ctx = pp.load_profiles(blat, list(bS), w3.n_classes, w3.batches, w3.bw)
    try:
        pp.enumerate(ctx, w3.kmax, w3.slo_us, w3.margin_permille)
        g2 = pp.pareto(ctx)
    finally:
        pp.free(ctx)
    assert np.array_equal(g1.points.view(np.uint8), g2.points.view(np.uint8))


@pytest.mark.parametrize("seed", range(24))
def test_random_models_with_ties(oracle_built, seed):
    rng = np.random.default_rng(9000 + seed)
    n = int(rng.integers(1, 6))
    C, B = int(rng.integers(1, 5)), int(rng.integers(1, 5))
    lats, Ss, Ms = [], [], []
    for _ in range(n):
        M = int(rng.integers(1, 300))
        hi = 4 if seed % 2 else 5000  # small values: exact ties and zero layers
        lats.append(rng.integers(0, hi, size=(C, M, B)).astype(np.uint32))
        Ss.append(rng.integers(1, 1 << 40, size=M).astype(np.uint64))
        Ms.append(M)
    N = int(rng.integers(1, min(Ms) + 1))
    _check(lats, Ss, N, int(rng.integers(0, C)), int(rng.integers(0, B)), f"random {seed}")


def test_one_layer_per_block_and_config5_models(oracle_built):
    w = config5(n_models=12)
    lats, Ss = [m.lat_us for m in w.models], [m.act_bytes for m in w.models]
    _check(lats, Ss, 10, 1, 0, "config 5 N=10")
    M = min(m.n_layers for m in w.models)
    bounds, _, _ = _check(lats, Ss, M, 0, 3, "config 5 N=M_min")
    small = [m for m in range(len(lats)) if lats[m].shape[1] == M]
    assert bounds[small[0]].tolist() == list(range(M + 1))


def test_errors():
    w = config3(n_blocks=None)
    lats, Ss = [w.models[0].lat_us], [w.models[0].act_bytes]
    M = w.models[0].n_layers
    for bad in [dict(n_blocks=M + 1), dict(n_blocks=0), dict(n_blocks=5, ref_class=4), dict(n_blocks=5, ref_batch=32)]:
        with pytest.raises(pp.PPipeError) as e:
            pp.prepartition(lats, Ss, **bad)
        assert e.value.code == -1, bad


def test_hand_worked_ties(oracle_built):
    """The hand-worked tie cases of tests/test_prepartition_pins.py on the GPU (ties take the layer)."""
    lat = np.array([[[3, 6], [2, 4], [2, 5], [5, 9]], [[30, 60], [20, 40], [20, 50], [50, 90]]], dtype=np.uint32)
    S = np.array([11, 12, 13, 14], np.uint64)
    b, _, _ = _check([lat], [S], 2, 0, 0, "tie [3,2,2,5]")
    assert b[0].tolist() == [0, 3, 4]
    b, _, _ = _check([lat], [S], 2, 0, 1, "no tie at b=2")
    assert b[0].tolist() == [0, 2, 4]
    one = np.array([1, 2, 1], np.uint32).reshape(1, 3, 1)
    b, _, _ = _check([one], [np.zeros(3, np.uint64)], 2, 0, 0, "tie [1,2,1]")
    assert b[0].tolist() == [0, 2, 3]
