"""Write tests/golden/f2_config4_oracle.json: the CPU oracle's F2 frontier (the
MILP-lossless per-stage-throughput frontier; F2-1..F2-4)
of config 4 (BASELINE.json configs[3]: one 500-layer CNN, 5 classes, batch 1-64, K <= 3),
as a SHA-256 of the records and of the per-segment counts plus the counts. Imports only
oracle/ and workloads/ (the literal all-pairs F2 definition in ppipe_oracle.c, f2_reduce).
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import run_oracle  # noqa: E402
from workloads import config4  # noqa: E402

w = config4()
t0 = time.time()
r = run_oracle(w, frontier=2)
sec = time.time() - t0
seg = np.diff(r.seg_offsets.astype(np.uint64)).astype("<u8")
out = {"config": 4, "frontier": "F2 (oracle_set_frontier(2))", "n_pts": int(r.points.shape[0]),
       "n_cand": int(r.n_candidates), "n_feas": int(r.n_feasible),
       "sha_pts": hashlib.sha256(r.points.tobytes()).hexdigest(),
       "sha_seg": hashlib.sha256(seg.tobytes()).hexdigest(), "oracle_sec": round(sec, 1),
       "threads": os.cpu_count()}
with open(os.path.join(ROOT, "tests", "golden", "f2_config4_oracle.json"), "w") as f:
    json.dump(out, f, indent=1)
print(out)
