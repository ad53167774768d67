"""Time ppipe_frontier_at (SLO sweep by truncation) after a config-5 enumeration."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2507_18748_b200 as pp  # noqa: E402
from workloads import config5  # noqa: E402

w = config5()
ctx = pp.load_workload(w)
pp.enumerate(ctx, w.kmax, w.slo_us, w.margin_permille)
g = pp.pareto(ctx, copy_to_host=False)
for rep in range(3):
    for sc in (0.9, 0.5, 0.1):
        t0 = time.perf_counter()
        f = pp.frontier_at(ctx, (w.slo_us * sc).astype(np.uint32), w.margin_permille, copy_to_host=False)
        print(f"rep {rep} scale {sc}: {1e3 * (time.perf_counter() - t0):.3f} ms wall, {f.n_points} points", flush=True)
pp.free(ctx)
