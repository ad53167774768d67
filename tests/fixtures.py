"""Hand-written fixtures for the pins (tests only)."""
from __future__ import annotations

import numpy as np

from workloads import ModelProfile, Workload

MIB = 1 << 20


def make_workload(lat_by_model, S_by_model, bw, batches, slo, margin=0, kmax=3, classes=None):
    """lat_by_model: list of arrays [C][M][B] (or [C][M] for a single batch)."""
    models = []
    for i, (lat, S) in enumerate(zip(lat_by_model, S_by_model)):
        lat = np.asarray(lat, dtype=np.uint32)
        if lat.ndim == 2:
            lat = lat[:, :, None]
        assert lat.shape[2] == len(batches), (lat.shape, batches)
        models.append(ModelProfile(f"fx{i}", lat, np.asarray(S, dtype=np.uint64)))
    C = models[0].lat_us.shape[0]
    bw = np.asarray(bw, dtype=np.uint32)
    if bw.ndim == 0:
        bw = np.full((C, C), int(bw), dtype=np.uint32)
    slo = np.asarray(slo if np.ndim(slo) else [slo] * len(models), dtype=np.uint32)
    return Workload(0, "fixture", classes or [f"k{i}" for i in range(C)],
                    np.asarray(batches, dtype=np.uint32), bw, models, slo, margin, kmax)


def t0(slo=200):
    """P0a: M=3, one class, batches {1,2}, Kmax=2 (SURVEY.md §8(c) hand-worked T0)."""
    lat = np.zeros((1, 3, 2), dtype=np.uint32)
    lat[0, :, 0] = [40, 20, 30]
    lat[0, :, 1] = [60, 30, 70]
    return make_workload([lat], [[1000, 250, 0]], 1000, [1, 2], slo, margin=0, kmax=2)


def t1():
    """P0b: exact duplicate (c=1 vs c=2) -> canonical c=1."""
    return make_workload([[[10, 0, 10]]], [[0, 0, 0]], 1000, [1], 10**6, margin=0, kmax=2)
