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


def test_hand_worked_ties_take_the_layer(oracle_built):
    """Hand-worked ties of the greedy rule ("as close as possible";
    ties include the layer, SPEC.md:138 / DESIGN.md reading of §5.2).

    t = [3, 2, 2, 5] (us), N = 2, total 12, target 12/2 = 6, compared as |N*acc - total|:
      block 1 starts with layer 0: acc = 3 (|6 - 12| = 6)
      layer 1: |2*5 - 12| = 2 <= 6  -> take, acc = 5
      layer 2: |2*7 - 12| = 2 <= 2  -> TIE, take, acc = 7
      layer 3 must stay for block 2 (one layer per remaining block) -> bounds [0, 3, 4]
    A strict "closer" rule would stop at [0, 2, 4]; a dropped tie rule fails here.
    Per-class / per-batch sums and the last layer's bytes follow by hand."""
    lat = np.array([[[3, 6], [2, 4], [2, 5], [5, 9]],        # class 0 (reference), b = 1, 2
                    [[30, 60], [20, 40], [20, 50], [50, 90]]], dtype=np.uint32)
    S = np.array([11, 12, 13, 14], np.uint64)
    b, blat, bS = prepartition_oracle(lat, S, 2, 0, 0)
    assert b.tolist() == [0, 3, 4]
    assert blat[0].tolist() == [[7, 15], [5, 9]]
    assert blat[1].tolist() == [[70, 150], [50, 90]]
    assert bS.tolist() == [13, 14]
    # the same tie at the reference batch b = 2: t = [6, 4, 5, 9], total 24, N*acc - total:
    #   acc 6 (|12-24| = 12); +4 -> |20-24| = 4 take; +5 -> |30-24| = 6 > 4 stop -> [0, 2, 4]
    b2, _, _ = prepartition_oracle(lat, S, 2, 0, 1)
    assert b2.tolist() == [0, 2, 4]
    # a tie at the very first comparison: t = [1, 2, 1], N = 2, total 4:
    #   acc 1 (|2-4| = 2); +2 -> |6-4| = 2 tie -> take; layer 2 left for block 2 -> [0, 2, 3]
    b3, blat3, _ = prepartition_oracle(_lat([1, 2, 1]), np.zeros(3, np.uint64), 2, 0, 0)
    assert b3.tolist() == [0, 2, 3] and blat3[0, :, 0].tolist() == [3, 1]
    # three blocks, tie in the middle block: t = [4, 2, 2, 2, 2], N = 3, total 12 (target 4):
    #   block 1: acc 4 (|12-12| = 0); +2 -> |18-12| = 6 > 0 stop -> layer 1 starts block 2
    #   block 2: acc 2 (|6-12| = 6); +2 -> |12-12| = 0 take; +2 -> 6 > 0 stop -> [0, 1, 3, 5]
    b4, _, _ = prepartition_oracle(_lat([4, 2, 2, 2, 2]), np.zeros(5, np.uint64), 3, 0, 0)
    assert b4.tolist() == [0, 1, 3, 5]
