"""Where does the e2e step time go? (config 5, N=1; wall clock per API call, synchronized)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2507_18748_b200 as pp
from workloads import make_config

w = make_config(5)
lat_h, S_h = [], []
for mp in w.models:
    lt = torch.empty(mp.lat_us.shape, dtype=torch.int32, pin_memory=True); lt.numpy().view(np.uint32)[...] = mp.lat_us
    st = torch.empty(mp.act_bytes.shape, dtype=torch.int64, pin_memory=True); st.numpy().view(np.uint64)[...] = mp.act_bytes
    lat_h.append(lt.numpy().view(np.uint32)); S_h.append(st.numpy().view(np.uint64))
ctx = pp.load_profiles(lat_h, S_h, w.n_classes, w.batches, w.bw, device=0)
def t(f):
    torch.cuda.synchronize(); a = time.perf_counter(); r = f(); torch.cuda.synchronize(); return (time.perf_counter() - a) * 1e3, r
for it in range(3):
    ms_u, _ = t(lambda: pp.update_profiles(ctx, lat_h, S_h))
    ms_e, _ = t(lambda: pp.enumerate(ctx, w.kmax, w.slo_us, w.margin_permille))
    ms_p, f = t(lambda: pp.pareto(ctx, copy_to_host=False))
    ms_e2, _ = t(lambda: pp.enumerate(ctx, w.kmax, w.slo_us, w.margin_permille))
    ms_pc, g = t(lambda: pp.pareto(ctx, copy_to_host=True))
    print(f"update {ms_u:.1f} ms | enumerate {ms_e:.2f} | pareto(dev) {ms_p:.1f} | pareto(copy) {ms_pc:.1f} | pts {g.n_points}", flush=True)
