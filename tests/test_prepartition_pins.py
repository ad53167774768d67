"""Pins of the oracle's greedy pre-partitioning (§5.2).

Each check comes from outside the oracle's own code: the worked examples of
SPEC.md:127-130, closed forms (one block; one layer per block; uniform layers),
per-block sums against numpy, and the balance bound that the paper's stopping
rule implies (a block that stopped by choice is within half of the next layer's
runtime of total/N).
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import prepartition_oracle


def _lat(ms):
    return np.asarray(ms, dtype=np.uint32).reshape(1, -1, 1)


def test_spec_example_forced_single_layer_blocks(oracle_built):
    b, blat, _ = prepartition_oracle(_lat([1000] * 10), np.arange(10, dtype=np.uint64), 10, 0, 0)
    assert b.tolist() == list(range(11))
    assert blat[0, :, 0].tolist() == [1000] * 10


def test_spec_example_9_1_1_9(oracle_built):
    b, blat, bS = prepartition_oracle(_lat([9000, 1000, 1000, 9000]), np.array([5, 6, 7, 8], np.uint64), 2, 0, 0)
    assert b.tolist() == [0, 2, 4]
    assert blat[0, :, 0].tolist() == [10000, 10000]
    assert bS.tolist() == [6, 8]  # output bytes of each block's last layer


def test_single_block_is_the_whole_model(oracle_built):
    rng = np.random.default_rng(1)
    lat = rng.integers(0, 500, size=(3, 37, 4)).astype(np.uint32)
    b, blat, bS = prepartition_oracle(lat, np.arange(37, dtype=np.uint64), 1, 1, 2)
    assert b.tolist() == [0, 37]
    assert np.array_equal(blat[:, 0, :], lat.astype(np.uint64).sum(axis=1))
    assert bS.tolist() == [36]


@pytest.mark.parametrize("M,N", [(12, 3), (40, 8), (60, 60), (100, 10)])
def test_uniform_layers_split_evenly(oracle_built, M, N):
    b, _, _ = prepartition_oracle(_lat([250] * M), np.zeros(M, np.uint64), N, 0, 0)
    assert b.tolist() == [q * (M // N) for q in range(N)] + [M]


@pytest.mark.parametrize("seed", range(40))
def test_random_models_cover_sum_and_balance(oracle_built, seed):
    rng = np.random.default_rng(500 + seed)
    C, M, B = int(rng.integers(1, 4)), int(rng.integers(1, 120)), int(rng.integers(1, 4))
    N = int(rng.integers(1, M + 1))
    lat = (rng.lognormal(5, 1.2, size=(C, M, B))).astype(np.uint32)
    if seed % 3 == 0:
        lat = rng.integers(0, 4, size=(C, M, B)).astype(np.uint32)  # many exact ties and zero layers
    S = rng.integers(1, 1 << 40, size=M).astype(np.uint64)
    rc, rb = int(rng.integers(0, C)), int(rng.integers(0, B))
    b, blat, bS = prepartition_oracle(lat, S, N, rc, rb)
    # coverage: N non-empty contiguous blocks over [0, M)
    assert b[0] == 0 and b[-1] == M and len(b) == N + 1
    assert (np.diff(b.astype(np.int64)) >= 1).all()
    # consistency: block latency = sum of member layers at every (class, batch); bytes of the last layer
    for q in range(N):
        assert np.array_equal(blat[:, q, :], lat[:, b[q]:b[q + 1], :].astype(np.uint64).sum(axis=1))
        assert bS[q] == S[b[q + 1] - 1]
    # balance (implied by "as close as possible to 1/N", not restated from the code): a
    # non-final block that stopped by choice (before the one-layer-per-block guard) is
    # within half a layer of total/N -- half the next layer if it undershoots, half its
    # last non-zero added layer if it overshoots -- unless its first layer alone exceeds
    # total/N, in which case every further layer it took has zero runtime
    t = lat[rc, :, rb].astype(np.int64)
    total = int(t.sum())
    for q in range(N - 1):
        i, j = int(b[q]), int(b[q + 1])
        if j >= M - (N - q - 1):
            continue  # stopped by the guard
        acc = int(t[i:j].sum())
        if N * int(t[i]) > total:
            assert acc == int(t[i]), (q, i, j)
            continue
        added = int(t[i + 1:j].max()) if j - i >= 2 else 0
        assert 2 * abs(N * acc - total) <= N * max(int(t[j]), added), (q, i, j)


def test_rejects_bad_block_counts(oracle_built):
    with pytest.raises(ValueError):
        prepartition_oracle(_lat([1, 2, 3]), np.zeros(3, np.uint64), 4, 0, 0)
    with pytest.raises(ValueError):
        prepartition_oracle(_lat([1, 2, 3]), np.zeros(3, np.uint64), 0, 0, 0)
