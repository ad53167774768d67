"""Write tests/golden/config5_oracle.json: the CPU oracle's frontier of every
config-5 model, as per-model SHA-256 digests plus counts.

Config 5 (BASELINE.json configs[4]): 1,000 synthetic CNN
profiles, M ~ U{400..826} (mean ~613), 5 classes, batch 1-64,
K <= 3, SLO = 5x the fastest class at b=1 with the 40%
margin deducted.

This script imports only ``oracle/`` (the arithmetic) and ``workloads/`` (the
seeded input recipe, no method arithmetic). Nothing here touches the CUDA
path. Per model m it stores:

* ``sha_pts``: SHA-256 of the model's frontier records (32-byte points, the
  canonical order of SURVEY.md §8(c) A17), exactly as the oracle emits them;
* ``sha_seg``: SHA-256 of the model's per-segment point counts (155 little-endian
  u64; segments in (K, class tuple) canonical order);
* ``n_pts``, ``n_cand``, ``n_feas``, and the oracle wall time ``sec``.

The run is resumable: progress is kept in ``<out>.partial`` after every model.
Usage: ``python scripts/golden_config5.py [--threads N] [--models lo:hi]``.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import run_oracle  # noqa: E402
from workloads import config5  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "config5_oracle.json")


def model_digest(res) -> dict:
    seg_counts = np.diff(res.seg_offsets.astype(np.uint64)).astype("<u8")
    return {
        "sha_pts": hashlib.sha256(res.points.tobytes()).hexdigest(),
        "sha_seg": hashlib.sha256(seg_counts.tobytes()).hexdigest(),
        "n_pts": int(res.points.shape[0]),
        "n_seg": int(seg_counts.shape[0]),
        "n_cand": int(res.n_candidates),
        "n_feas": int(res.n_feasible),
    }


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=0, help="oracle threads (0 = all host cores)")
    ap.add_argument("--models", default="0:1000")
    ap.add_argument("--out", default=OUT)
    a = ap.parse_args()
    lo, hi = (int(x) for x in a.models.split(":"))
    w = config5(n_models=1000)
    partial = a.out + ".partial"
    state = {"models": {}}
    if os.path.exists(partial):
        with open(partial) as f:
            state = json.load(f)
    threads = a.threads or os.cpu_count()
    state.update({
        "config": 5,
        "workload": "config5(n_models=1000): 1,000 x M~U{400..826}, 5 classes, b 1..64, K<=3, margin 400",
        "generator": "workloads.generate.config5, seeds 250718748 + 5000 + model (numpy PCG64)",
        "oracle": "oracle/ppipe_oracle.c oracle_run (nested loops, direct sums, sort + strict staircase)",
        "record": "32-byte point (model u32, cut u16[2], K u8, cls u8[3], batch u16, reserved u16, e2e u32, stage u32[3])",
        "threads": threads,
        "host_cores": os.cpu_count(),
    })
    for m in range(lo, hi):
        key = str(m)
        if key in state["models"]:
            continue
        t0 = time.time()
        res = run_oracle(w, model_lo=m, model_hi=m + 1, threads=threads)
        d = model_digest(res)
        d["sec"] = round(time.time() - t0, 3)
        d["M"] = w.models[m].n_layers
        state["models"][key] = d
        with open(partial + ".tmp", "w") as f:
            json.dump(state, f)
        os.replace(partial + ".tmp", partial)
        print(f"model {m} M={d['M']} pts={d['n_pts']} feas={d['n_feas']} {d['sec']}s", flush=True)
    if len(state["models"]) == 1000:
        ms = state["models"]
        state["total"] = {
            "n_pts": sum(v["n_pts"] for v in ms.values()),
            "n_cand": sum(v["n_cand"] for v in ms.values()),
            "n_feas": sum(v["n_feas"] for v in ms.values()),
            "oracle_sec": round(sum(v["sec"] for v in ms.values()), 1),
        }
        ordered = dict(state)
        ordered["models"] = {str(i): ms[str(i)] for i in range(1000)}
        with open(a.out, "w") as f:
            json.dump(ordered, f, indent=0)
        print("wrote", a.out, state["total"])


if __name__ == "__main__":
    main()
