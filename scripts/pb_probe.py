"""Time ppipe_pareto_pb on a config (device phases via ppipe_phase_ms)."""
import argparse
import json
import sys
import time

sys.path.insert(0, ".")
import paper_2507_18748_b200 as pp  # noqa: E402
from workloads import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--models", type=int, default=0)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
kw = {"n_models": a.models} if a.models else {}
w = make_config(a.config, **kw)
ctx = pp.load_workload(w)
for r in range(a.reps):
    t = time.time()
    f = pp.pareto_pb(ctx, w.kmax, w.slo_us, w.margin_permille, copy_to_host=False)
    dt = time.time() - t
    print(json.dumps(dict(rep=r, wall_ms=dt * 1e3, phase_ms=ctx.phase_ms(), n_cand=f.n_candidates,
                          n_feas=f.n_feasible, n_surv=f.n_survivors, n_pts=f.n_points,
                          launches=ctx.launch_count())), flush=True)
pp.free(ctx)
