"""Where does the e2e step time go? (config 5, N=1): the async-upload step's device phases
(ppipe_phase_ms: [0] upload + validate + pack + score3a chunks, [1] score3b + score12,
[2] frontier, [3] merge) and the wall time of each API call."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2507_18748_b200 as pp  # noqa: E402
from workloads import make_config  # noqa: E402

w = make_config(5)
lat_h, S_h = [], []
if "--separate" in sys.argv:  # one pinned allocation per model array
    for mp in w.models:
        lt = torch.empty(mp.lat_us.shape, dtype=torch.int32, pin_memory=True)
        lt.numpy().view(np.uint32)[...] = mp.lat_us
        st = torch.empty(mp.act_bytes.shape, dtype=torch.int64, pin_memory=True)
        st.numpy().view(np.uint64)[...] = mp.act_bytes
        lat_h.append(lt.numpy().view(np.uint32))
        S_h.append(st.numpy().view(np.uint64))
else:  # one pinned buffer per kind, sliced per model (as bench.py)
    lat_all = torch.empty(sum(mp.lat_us.size for mp in w.models), dtype=torch.int32, pin_memory=True)
    S_all = torch.empty(sum(mp.act_bytes.size for mp in w.models), dtype=torch.int64, pin_memory=True)
    la, sa = lat_all.numpy().view(np.uint32), S_all.numpy().view(np.uint64)
    ol = os_ = 0
    for mp in w.models:
        lat_h.append(la[ol:ol + mp.lat_us.size].reshape(mp.lat_us.shape))
        lat_h[-1][...] = mp.lat_us
        S_h.append(sa[os_:os_ + mp.act_bytes.size].reshape(mp.act_bytes.shape))
        S_h[-1][...] = mp.act_bytes
        ol += mp.lat_us.size
        os_ += mp.act_bytes.size
ctx = pp.load_profiles(lat_h, S_h, w.n_classes, w.batches, w.bw, device=0)
for it in range(4):
    torch.cuda.synchronize()
    a = time.perf_counter()
    pp.update_profiles_async(ctx, lat_h, S_h)
    b = time.perf_counter()
    pp.enumerate(ctx, w.kmax, w.slo_us, w.margin_permille)
    c = time.perf_counter()
    g = pp.pareto(ctx, copy_to_host=True, zero_copy=True)
    d = time.perf_counter()
    ph = ctx.phase_ms()
    print(f"e2e step {1e3 * (d - a):.1f} ms: update_async {1e3 * (b - a):.2f}, enumerate (host) {1e3 * (c - b):.2f}, "
          f"pareto+D2H {1e3 * (d - c):.1f} | device phases {[round(x, 2) for x in ph]} | pts {g.n_points}", flush=True)
for it in range(2):
    torch.cuda.synchronize()
    a = time.perf_counter()
    pp.enumerate(ctx, w.kmax, w.slo_us, w.margin_permille)
    g = pp.pareto(ctx, copy_to_host=True, zero_copy=True)
    d = time.perf_counter()
    print(f"resident step + D2H {1e3 * (d - a):.1f} ms | phases {[round(x, 2) for x in ctx.phase_ms()]}", flush=True)
pp.free(ctx)
