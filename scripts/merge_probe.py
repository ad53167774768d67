"""Time ppipe_merge_shards: W shard-mode contexts of config 5 on one GPU (the NCCL merge's
assembly without the all-gathers). usage: python scripts/merge_probe.py [W] [models]"""
import sys
import time

sys.path.insert(0, ".")
import paper_2507_18748_b200 as pp  # noqa: E402
from workloads import config5  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 4
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
w = config5(n_models=n)
ctxs = [pp.load_workload(w, rank=r, world=W) for r in range(W)]
for rep in range(3):
    for c in ctxs:
        pp.enumerate(c, w.kmax, w.slo_us, w.margin_permille)
        pp.pareto(c, copy_to_host=False)
    t0 = time.perf_counter()
    g = pp.merge_shards(ctxs, copy_to_host=False)
    dt = (time.perf_counter() - t0) * 1e3
    print(f"rep {rep}: merge {dt:.3f} ms wall, device {ctxs[0].phase_ms()[3]:.3f} ms, {g.n_points} points, "
          f"launches {ctxs[0].launch_count()}", flush=True)
for c in ctxs:
    pp.free(c)
