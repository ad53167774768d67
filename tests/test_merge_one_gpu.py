"""The multi-GPU frontier merge exercised on ONE GPU.

W shard-mode contexts (rank r of W, no NCCL id) each enumerate their equal-weight
first-cut-row shard and reduce it to a local frontier; ppipe_merge_shards then runs
the library's own merge -- the code the NCCL path runs after its two all-gathers:
per-rank counters, rank-ordered pieces, re-reduction of the models straddling a rank
boundary, assembly, CSR -- with the all-gathers replaced by device copies. The merged
frontier must equal the oracle's (configs 3 and 4) and the one-rank result (a config-5
slice) byte for byte.
"""
from __future__ import annotations

import numpy as np
import pytest

import paper_2507_18748_b200 as pp
from oracle import run_oracle
from tests.helpers import assert_same_result
from workloads import config3, config4, config5

pytestmark = pytest.mark.gpu


def _merged(w, world):
    ctxs = [pp.load_workload(w, rank=r, world=world) for r in range(world)]
    try:
        for c in ctxs:
            pp.enumerate(c, w.kmax, w.slo_us, w.margin_permille)
            pp.pareto(c, copy_to_host=False)
        return pp.merge_shards(ctxs)
    finally:
        for c in ctxs:
            pp.free(c)


@pytest.mark.parametrize("world", [2, 3, 5, 8])
def test_merge_config3_vs_oracle(oracle_built, world):
    w = config3()
    assert_same_result(_merged(w, world), run_oracle(w), f"config 3 merged from {world} shards")


@pytest.mark.parametrize("world", [2, 3, 5, 8])
def test_merge_config4_vs_oracle(oracle_built, world):
    """One model split into W shards: every rank boundary cuts through it."""
    w = config4()
    assert_same_result(_merged(w, world), run_oracle(w), f"config 4 merged from {world} shards")


@pytest.mark.parametrize("world", [2, 3, 5, 8])
def test_merge_config5_slice_vs_one_rank(world):
    w = config5(n_models=40)
    one = pp.run(w)
    g = _merged(w, world)
    assert g.n_candidates == one.n_candidates and g.n_feasible == one.n_feasible
    assert np.array_equal(g.points.view(np.uint8), one.points.view(np.uint8))
    assert np.array_equal(g.seg_offsets, one.seg_offsets)


def test_merge_with_more_ranks_than_rows(oracle_built):
    """Ranks without rows (tiny model, many ranks) contribute nothing and still merge."""
    w = config3(n_models=2)
    assert_same_result(_merged(w, 40), run_oracle(w), "config 3 (2 models) merged from 40 shards")


def test_merge_rejects_mismatched_shards():
    w = config3(n_models=3)
    a = pp.load_workload(w, rank=0, world=2)
    b = pp.load_workload(w, rank=0, world=2)
    try:
        for c in (a, b):
            pp.enumerate(c, w.kmax, w.slo_us, w.margin_permille)
            pp.pareto(c, copy_to_host=False)
        with pytest.raises(pp.PPipeError) as e:
            pp.merge_shards([a, b])
        assert e.value.code == -1 and "shard 1 is rank 0 of 2" in str(e.value)
    finally:
        pp.free(a)
        pp.free(b)
