"""Seeded synthetic inputs shaped like the paper's workloads.

Recipe:

* Per-layer latency, reference class (L4-like) at batch 1:
  ``x_l ~ LogNormal(0, 1)`` normalised to a model total ``T1_ref``; ``T1_ref``
  is log-uniform in [4.68, 33.12] ms so that the default SLO ``5 * T1`` spans
  the paper's 23.4-165.6 ms (§7.1 Setup).
* Class ``k`` per-layer ratio ``rho_k(l) = ramp_k(l/(M-1)) * LogNormal(0, .15)``
  renormalised so the model total is ``R_k * T1_ref``. P4/L4 ramps from ~1.7
  on early layers to much higher on late layers, P4/V100 the other way round
  (§2 Fig. 3); P4/L4 totals 3.0-7.9x.
* Batch: ``lat(l,k,b) = round_half_up(x_l rho_k(l) (a + (1-a) b))`` with
  ``a ~ U[0.2, 0.9]`` per (layer, class): monotone in b, amortising per
  sample. Integer microseconds, so some layers round to 0 us.
* Feature maps: CNN-like schedule (spatial halves, channels double per stage),
  adjacent-layer oscillation up to ~12x, fp32 size in
  [0.1, 50] MiB at batch 1, halved for the fp16 wire
  (§6).
* Bandwidth: nominal 50 Gbps (L4 / V100 / P4 / X hosts) or 32 Gbps (T4 hosts)
  per Table 1; effective = 1/5;
  pair value = min of the two ends. Unit: bits/us.
* SLO: 5x the whole-model latency on the fastest class at batch 1
  (reading A16); margin 40%.

Seeds: ``250718748 + 1000 * config + model`` (numpy PCG64).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

SEED_BASE = 250718748
MIB = 1 << 20
KIB = 1 << 10

CONFIG_NAMES = {
    1: "toy 8-layer CNN, 2 GPU classes, batch {1,2,4}, K<=2 partitions, SLO 200 ms",
    2: "ResNet-50 block-level profile, 3 GPU classes, batch 1-32, K<=3, SLO 200 ms",
    3: "18-CNN suite shaped like the paper's workloads, 4 GPU classes, batch 1-32, K<=3",
    4: "fine-grained layer cuts of a deep CNN (~500 layers), 5 GPU classes, batch 1-64, K<=3",
    5: "8-GPU scaling sweep: 1,000 synthetic CNN profiles x 5 classes x batch 1-64, K<=3",
}

# name -> (total latency ratio vs L4-like, ramp start, ramp end, nominal Gbps)
CLASS_LIBRARY = {
    "V100": (0.8, 0.15, 1.8, 50),
    "L4": (1.0, 1.0, 1.0, 50),
    "T4": (2.0, 1.4, 2.6, 32),
    "P4": (5.0, 1.7, 9.0, 50),
    "X": (0.5, 1.0, 1.0, 50),
}


@dataclass
class ModelProfile:
    name: str
    lat_us: np.ndarray  # uint32 [C][M][B]
    act_bytes: np.ndarray  # uint64 [M], on-wire bytes of layer l's output at batch 1

    @property
    def n_layers(self) -> int:
        return int(self.lat_us.shape[1])


@dataclass
class Workload:
    config: int
    name: str
    classes: List[str]
    batches: np.ndarray  # uint32 [B], strictly increasing
    bw: np.ndarray  # uint32 [C][C] bits/us (sender, receiver)
    models: List[ModelProfile]
    slo_us: np.ndarray  # uint32 [n_models]
    margin_permille: int = 400
    kmax: int = 3
    meta: dict = field(default_factory=dict)

    @property
    def n_classes(self) -> int:
        return len(self.classes)

    @property
    def n_batches(self) -> int:
        return int(self.batches.shape[0])

    def subset(self, model_ids: Sequence[int]) -> "Workload":
        ids = list(model_ids)
        return Workload(self.config, self.name + f" [models {ids[:4]}{'...' if len(ids) > 4 else ''}]",
                        list(self.classes), self.batches.copy(), self.bw.copy(),
                        [self.models[i] for i in ids], self.slo_us[ids].copy(),
                        self.margin_permille, self.kmax, dict(self.meta))


def _bw_matrix(classes: Sequence[str]) -> np.ndarray:
    eff = [CLASS_LIBRARY[c][3] * 1000 // 5 for c in classes]  # Gbps -> bits/us, /5 effective
    C = len(classes)
    bw = np.zeros((C, C), dtype=np.uint32)
    for i in range(C):
        for j in range(C):
            bw[i, j] = min(eff[i], eff[j])
    return bw


def _round_half_up(x: np.ndarray) -> np.ndarray:
    return np.floor(x + 0.5)


def _layer_latencies(rng: np.random.Generator, M: int, classes: Sequence[str],
                     batches: np.ndarray, t1_ref_us: float) -> np.ndarray:
    x = rng.lognormal(0.0, 1.0, size=M)
    x *= t1_ref_us / x.sum()
    u = np.linspace(0.0, 1.0, M) if M > 1 else np.zeros(1)
    C, B = len(classes), len(batches)
    lat = np.zeros((C, M, B), dtype=np.float64)
    for k, cname in enumerate(classes):
        R, r0, r1, _ = CLASS_LIBRARY[cname]
        ramp = r0 ** (1.0 - u) * r1 ** u
        rho = ramp * rng.lognormal(0.0, 0.15, size=M)
        rho *= R * x.sum() / (x * rho).sum()
        alpha = rng.uniform(0.2, 0.9, size=M)
        base = x * rho
        for bi, b in enumerate(batches):
            lat[k, :, bi] = base * (alpha + (1.0 - alpha) * float(b))
    return _round_half_up(lat).astype(np.uint32)


def _act_bytes(rng: np.random.Generator, M: int) -> np.ndarray:
    stages = 5
    base = np.exp(rng.uniform(np.log(4 * MIB), np.log(24 * MIB)))
    stage = np.minimum((np.arange(M) * stages) // max(M, 1), stages - 1)
    osc = np.exp(rng.uniform(np.log(1 / 3.5), np.log(3.5), size=M))
    fp32 = np.clip(base * 0.5 ** stage * osc, 0.1 * MIB, 50 * MIB)
    return (np.floor(fp32 / 2.0)).astype(np.uint64)


def _default_slo(lat: np.ndarray, batches: np.ndarray) -> int:
    # 5x whole-model latency on the fastest class at batch 1.
    b1 = int(np.nonzero(batches == 1)[0][0])
    totals = lat[:, :, b1].astype(np.int64).sum(axis=1)
    return int(5 * totals.min())


def config1() -> Workload:
    """Hand-written toy. Not generated."""
    H1 = np.array([4000, 6000, 0, 9000, 7000, 5000, 8000, 1000], dtype=np.int64)
    L1 = np.array([6000, 10000, 0, 18000, 21000, 15000, 24000, 6000], dtype=np.int64)
    batches = np.array([1, 2, 4], dtype=np.uint32)
    lat = np.zeros((2, 8, 3), dtype=np.uint32)
    for k, row in enumerate((H1, L1)):
        lat[k, :, 0] = row
        lat[k, :, 1] = row * 16 // 10
        lat[k, :, 2] = row * 28 // 10
    S = np.array([2 * MIB, 8 * MIB, 8 * MIB, 1 * MIB, 4 * MIB, 512 * KIB, 256 * KIB, 4 * KIB], dtype=np.uint64)
    bw = np.full((2, 2), 10000, dtype=np.uint32)
    return Workload(1, CONFIG_NAMES[1], ["H", "L"], batches, bw, [ModelProfile("toy8", lat, S)],
                    np.array([200000], dtype=np.uint32), 400, 2)


def config2() -> Workload:
    """ResNet-50 at block granularity: stem, 16 bottlenecks (3+4+6+3), head."""
    rng = np.random.Generator(np.random.PCG64(SEED_BASE + 1000 * 2 + 0))
    classes = ["L4", "T4", "P4"]
    batches = np.arange(1, 33, dtype=np.uint32)
    M = 18
    lat = _layer_latencies(rng, M, classes, batches, 8000.0)
    elems = [64 * 56 * 56] + [256 * 56 * 56] * 3 + [512 * 28 * 28] * 4 + \
            [1024 * 14 * 14] * 6 + [2048 * 7 * 7] * 3 + [1000]
    S = np.array([2 * e for e in elems], dtype=np.uint64)  # fp16 on the wire
    return Workload(2, CONFIG_NAMES[2], classes, batches, _bw_matrix(classes),
                    [ModelProfile("resnet50-blocks", lat, S)], np.array([200000], dtype=np.uint32), 400, 3)


def _prepartition_input_step(lat: np.ndarray, S: np.ndarray, n_blocks: int, ref_class: int, b1: int):
    """INPUT STEP (not the method under test): build config 3's block profiles by
    greedy equal-runtime grouping (§5.2).

    Extend the current block while doing so brings its batch-1 runtime on the
    reference class closer to total/N (ties include the layer), leaving at least
    one layer per remaining block (SPEC.md:117-149 guard). Block latency = sum of
    member layers per (class, batch); block output bytes = last member's.
    """
    M = lat.shape[1]
    t = lat[ref_class, :, b1].astype(np.int64)
    target = t.sum() / n_blocks
    bounds = [0]
    i = 0
    for blk in range(n_blocks - 1):
        remaining_blocks = n_blocks - blk - 1
        j = i + 1
        acc = t[i]
        while j < M - remaining_blocks:
            if abs(acc + t[j] - target) <= abs(acc - target):
                acc += t[j]
                j += 1
            else:
                break
        bounds.append(j)
        i = j
    bounds.append(M)
    C, _, B = lat.shape
    blat = np.zeros((C, n_blocks, B), dtype=np.uint64)
    bS = np.zeros(n_blocks, dtype=np.uint64)
    for q in range(n_blocks):
        blat[:, q, :] = lat[:, bounds[q]:bounds[q + 1], :].astype(np.uint64).sum(axis=1)
        bS[q] = S[bounds[q + 1] - 1]
    return blat.astype(np.uint32), bS, bounds


def config3(n_models: int = 18, n_blocks: Optional[int] = 10) -> Workload:
    """18 CNN-like models pre-partitioned into n_blocks blocks on the L4-like class at
    batch 1; n_blocks=None gives the layer-level models ("3L")."""
    classes = ["V100", "L4", "T4", "P4"]
    batches = np.arange(1, 33, dtype=np.uint32)
    models, slos = [], []
    for m in range(n_models):
        rng = np.random.Generator(np.random.PCG64(SEED_BASE + 1000 * 3 + m))
        M = int(rng.integers(150, 1077))
        t1 = float(np.exp(rng.uniform(np.log(4680.0), np.log(33120.0))))
        lat = _layer_latencies(rng, M, classes, batches, t1)
        S = _act_bytes(rng, M)
        slo = _default_slo(lat, batches)
        if n_blocks is None:
            models.append(ModelProfile(f"cnn{m:02d}", lat, S))
        else:
            blat, bS, _ = _prepartition_input_step(lat, S, n_blocks, classes.index("L4"), 0)
            models.append(ModelProfile(f"cnn{m:02d}-N{n_blocks}", blat, bS))
        slos.append(slo)
    return Workload(3, CONFIG_NAMES[3], classes, batches, _bw_matrix(classes), models,
                    np.array(slos, dtype=np.uint32), 400, 3)


def _deep_model(config: int, m: int, M: Optional[int], classes, batches, m_range=(400, 826)):
    rng = np.random.Generator(np.random.PCG64(SEED_BASE + 1000 * config + m))
    if M is None:
        M = int(rng.integers(m_range[0], m_range[1] + 1))
    t1 = float(np.exp(rng.uniform(np.log(4680.0), np.log(33120.0))))
    lat = _layer_latencies(rng, M, classes, batches, t1)
    S = _act_bytes(rng, M)
    return ModelProfile(f"cnn{config}-{m:04d}-M{M}", lat, S), _default_slo(lat, batches)


CLASSES5 = ["V100", "L4", "T4", "P4", "X"]


def config4() -> Workload:
    batches = np.arange(1, 65, dtype=np.uint32)
    mp, slo = _deep_model(4, 0, 500, CLASSES5, batches)
    return Workload(4, CONFIG_NAMES[4], list(CLASSES5), batches, _bw_matrix(CLASSES5), [mp],
                    np.array([slo], dtype=np.uint32), 400, 3)


def config5(n_models: int = 1000, model_ids: Optional[Sequence[int]] = None) -> Workload:
    batches = np.arange(1, 65, dtype=np.uint32)
    ids = list(range(n_models)) if model_ids is None else list(model_ids)
    models, slos = [], []
    for m in ids:
        mp, slo = _deep_model(5, m, None, CLASSES5, batches)
        models.append(mp)
        slos.append(slo)
    w = Workload(5, CONFIG_NAMES[5], list(CLASSES5), batches, _bw_matrix(CLASSES5), models,
                 np.array(slos, dtype=np.uint32), 400, 3)
    w.meta["model_ids"] = ids
    return w


def make_config(config: int, **kw) -> Workload:
    return {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}[config](**kw)


def random_tiny(seed: int, max_layers: int = 8, max_classes: int = 3, max_batches: int = 4,
                n_models: int = 1, kmax: Optional[int] = None) -> Workload:
    """Random tiny fuzz input: zero-latency layers, ties and batch-non-monotone
    latencies included on purpose (SURVEY.md §4 test layer 2, readings A12/A13)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    C = int(rng.integers(1, max_classes + 1))
    B = int(rng.integers(1, max_batches + 1))
    batches = np.sort(rng.choice(np.arange(1, 9), size=B, replace=False)).astype(np.uint32)
    models, slos = [], []
    for m in range(n_models):
        M = int(rng.integers(1, max_layers + 1))
        lat = rng.integers(0, 12, size=(C, M, B)).astype(np.uint32) * 5  # coarse -> many ties
        lat[rng.random(size=lat.shape) < 0.2] = 0
        for k in range(C):
            for bi in range(B):
                if lat[k, :, bi].sum() == 0:
                    lat[k, int(rng.integers(0, M)), bi] = 5
        S = (rng.integers(0, 4, size=M) * 250).astype(np.uint64)
        models.append(ModelProfile(f"tiny{seed}-{m}", lat, S))
        slos.append(int(rng.integers(20, 400)))
    bw = rng.choice(np.array([500, 1000, 2000], dtype=np.uint32), size=(C, C)).astype(np.uint32)
    margin = int(rng.choice([0, 100, 400]))
    K = int(rng.integers(1, 4)) if kmax is None else kmax
    return Workload(0, f"tiny seed {seed}", [f"c{i}" for i in range(C)], batches, bw, models,
                    np.array(slos, dtype=np.uint32), margin, K)
