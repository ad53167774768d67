#!/usr/bin/env python
"""Benchmark: pipeline-plan candidates scored per second (BASELINE.json metric).

One step = one pass of the whole hot path over
config 5 (1,000 synthetic CNN profiles x 5 classes x batch 1-64, K <= 3):
pack -> score + fold -> frontier pass (-> NCCL all-gather + final pass for N > 1),
inputs resident in HBM. Launch: `python bench.py --gpus 1 --steps K --warmup W`,
or under torchrun for N > 1 (one process per GPU). Prints ONE JSON line (rank 0).

`--impl reference` times the CPU oracle (oracle/, the correctness reference of
this build) on the box's host cores on bounded samples of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "pipeline-plan candidates scored/sec at 1/2/4/8 B200; % of INT32 issue roofline"
UNIT = "candidates/s"
SM_COUNT = 148
ISSUE_LANES_PER_CLK_PER_SM = 128  # 4 SMSPs x 1 warp-instruction/clk x 32 lanes: integer issue ceiling


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def _host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""

    def __init__(self):
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self, gpus):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9 or not f[0].isdigit() or int(f[0]) not in gpus:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        os.unlink(self.path)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_baseline(cfg: int, target_s: float = 12.0, cap_s: float = 30.0):
    """The oracle as it stands, on host cores, over whole config models until ~target_s."""
    from oracle import run_oracle
    from workloads import config5, make_config
    threads = _host_threads()
    cand, t_tot, used = 0, 0.0, []
    m = 0
    while t_tot < target_s:
        w = config5(model_ids=[m]) if cfg == 5 else make_config(cfg)
        t0 = time.perf_counter()
        r = run_oracle(w, threads=threads)
        dt = time.perf_counter() - t0
        cand += r.n_candidates
        t_tot += dt
        used.append(m)
        m += 1
        if cfg != 5 or t_tot > cap_s:
            break
    return {"value": cand / t_tot, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"config {cfg} model(s) {used[0]}..{used[-1]} in full ({cand} candidates, {t_tot:.1f} s)"}


def oracle_rate(w, threads: int, target_s: float = 3.0):
    """The oracle's candidates/s on a workload: in full if that takes under ~target_s,
    else on a calibrated range of model 0's first-cut rows (row 0 = the K = 1 candidates)."""
    from oracle import run_oracle
    t0 = time.perf_counter()
    if len(w.models) > 1 or w.models[0].n_layers < 64:
        r = run_oracle(w, threads=threads)
        return r.n_candidates / (time.perf_counter() - t0), "in full"
    M = w.models[0].n_layers
    rows = 4
    while True:
        t0 = time.perf_counter()
        r = run_oracle(w, threads=threads, row_lo=1, row_hi=1 + rows)
        dt = time.perf_counter() - t0
        if dt > target_s / 4 or rows >= M - 1:
            break
        rows = min(M - 1, rows * 2)
    if rows < M - 1:
        rows = max(1, min(M - 1, int(rows * target_s / max(dt, 1e-3))))
        t0 = time.perf_counter()
        r = run_oracle(w, threads=threads, row_lo=1, row_hi=1 + rows)
        dt = time.perf_counter() - t0
    return r.n_candidates / dt, f"first-cut rows [1, {1 + rows}) of {M - 1}"


def per_config_block(pp, local_rank: int, steps: int = 5, with_oracle: bool = True) -> dict:
    """Configs 1-4 (BASELINE.json configs[0..3]): device-timed candidates/s of one
    enumerate + pareto step (inputs resident, CUDA events on the library stream), frontier
    points, and the oracle's single-thread and all-core rates on the host."""
    import torch
    from workloads import CONFIG_NAMES, make_config
    threads = _host_threads()
    out = {}
    for cfg in (1, 2, 3, 4):
        w = make_config(cfg)
        ctx = pp.load_workload(w, device=local_rank)
        try:
            st = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local_rank))
            for _ in range(2):
                pp.enumerate(ctx, w.kmax, w.slo_us, w.margin_permille)
                f = pp.pareto(ctx, copy_to_host=False)
            ms = []
            for _ in range(steps):
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(st)
                pp.enumerate(ctx, w.kmax, w.slo_us, w.margin_permille)
                f = pp.pareto(ctx, copy_to_host=False)
                e1.record(st)
                e1.synchronize()
                ms.append(e0.elapsed_time(e1))
        finally:
            pp.free(ctx)
        med = statistics.median(ms)
        d = {"workload": CONFIG_NAMES[cfg], "candidates": f.n_candidates, "feasible": f.n_feasible,
             "frontier_points": f.n_points, "ms_per_step": med, "candidates_per_s": f.n_candidates / (med / 1e3)}
        if with_oracle:
            r1, s1 = oracle_rate(w, 1)
            rn, sn = oracle_rate(w, threads)
            d["oracle_1_thread"] = {"candidates_per_s": r1, "sample": s1}
            d["oracle_all_cores"] = {"candidates_per_s": rn, "threads": threads, "sample": sn}
        out[f"config {cfg}"] = d
    out["timing"] = (f"median of {steps} device-timed enumerate + pareto steps per config (2 warm-up), inputs "
                     "resident; oracle rates on the host (single thread and all cores, in full or on a "
                     "calibrated first-cut-row range of the model)")
    return out


def score_profile(config: int):
    """ncu counters of the score kernels of one config-5 step of this build
    (profiles/r2_score_ncu.json, written by scripts/profile_score.py from an ncu --set full
    capture): executed warp-instructions and DRAM bytes per step."""
    path = os.path.join(ROOT, "profiles", "r2_score_ncu.json")
    try:
        pj = json.load(open(path))
    except Exception:
        return None
    if int(pj.get("config", 5)) != config:
        return None
    return pj


def run_reference(args):
    """--impl reference: the CPU oracle on bounded samples of the same workload."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import run_oracle
    from workloads import CONFIG_NAMES, config5, make_config
    threads = _host_threads()
    w = config5(model_ids=[0]) if args.config == 5 else make_config(args.config)
    M = w.models[0].n_layers
    # calibrate a first-cut row range of model 0 to ~4 s per step
    rows = 8
    while True:
        t0 = time.perf_counter()
        r = run_oracle(w, threads=threads, row_lo=1, row_hi=1 + rows)
        dt = time.perf_counter() - t0
        if dt > 1.0 or rows >= M - 1:
            break
        rows = min(M - 1, rows * 2)
    rows = max(1, min(M - 1, int(rows * 4.0 / max(dt, 1e-3))))
    times, cands = [], []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        r = run_oracle(w, threads=threads, row_lo=1, row_hi=1 + rows)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
            cands.append(r.n_candidates)
    value = sum(cands) / sum(times)
    sample = (f"config {args.config} model 0 first-cut rows [1, {1 + rows}) of {M - 1}: "
              f"{cands[0]} candidates per step")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * sum(times) / len(times),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic", "config": {"workload": f"config {args.config}: {CONFIG_NAMES[args.config]}",
                                            "sample": sample},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit_line(line)
    return 0


_JSON_OUT = None


def emit_line(line: dict) -> None:
    """The one JSON line on stdout (rank 0). Everything else that reaches fd 1 -- NCCL's
    version banner, library prints -- was redirected to stderr by main()."""
    out = _JSON_OUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the SLO-sweep (frontier_at) measurement")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-f2", action="store_true", help="skip the F2 (MILP-lossless frontier) measurement")
    ap.add_argument("--no-pb", action="store_true", help="skip the per-stage batch (App. A.1) measurement")
    ap.add_argument("--models", type=int, default=None, help="config 5 only: first N models (profiling)")
    ap.add_argument("--margin", type=int, default=None, help="override margin_permille (experiments)")
    ap.add_argument("--no-per-config", action="store_true", help="skip the configs 1-4 block")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2507_18748_b200 as pp
    from workloads import make_config

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"warning: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    from paper_2507_18748_b200.build import build
    if rank == 0:
        build()
    if world > 1:
        dist.barrier()

    w = make_config(args.config, **({"n_models": args.models} if args.models and args.config == 5 else {}))
    if args.margin is not None:
        w.margin_permille = args.margin
    nccl_id = None
    if world > 1:
        t = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            t.copy_(torch.frombuffer(bytearray(pp.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(t, 0)
        nccl_id = bytes(t.cpu().numpy().tobytes())

    # pinned host copies of the inputs (the e2e leg copies them H2D every step): one
    # page-locked buffer per kind, sliced per model (the library merges the copies of
    # adjacent models)
    lat_all = torch.empty(sum(mp.lat_us.size for mp in w.models), dtype=torch.int32, pin_memory=True)
    S_all = torch.empty(sum(mp.act_bytes.size for mp in w.models), dtype=torch.int64, pin_memory=True)
    lat_np, S_np = lat_all.numpy().view(np.uint32), S_all.numpy().view(np.uint64)
    lat_h, S_h = [], []
    ol = os_ = 0
    for mp in w.models:
        lt = lat_np[ol:ol + mp.lat_us.size].reshape(mp.lat_us.shape)
        lt[...] = mp.lat_us
        st = S_np[os_:os_ + mp.act_bytes.size].reshape(mp.act_bytes.shape)
        st[...] = mp.act_bytes
        ol += mp.lat_us.size
        os_ += mp.act_bytes.size
        lat_h.append(lt)
        S_h.append(st)

    ctx = pp.load_profiles(lat_h, S_h, w.n_classes, w.batches, w.bw, rank=rank, world=world, device=local_rank,
                           nccl_id=nccl_id)
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def step(copy=False):
        pp.enumerate(ctx, w.kmax, w.slo_us, w.margin_permille)
        # e2e: the frontier lands in the context's page-locked buffer and is read in place
        return pp.pareto(ctx, copy_to_host=copy, zero_copy=copy)

    for _ in range(args.warmup):
        f = step()

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    sampler = ClockSampler()
    barrier()
    if rank == 0:
        sampler.start()
        time.sleep(0.3)
    barrier()
    step_ms, kern_ms, launches, phases = [], [], 0, []
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()  # L2 flush between timed steps (not timed)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        f = step()
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        ph = ctx.phase_ms()
        phases.append(ph)
        kern_ms.append(ph[1])
        launches += ctx.launch_count()
    barrier()
    clocks = sampler.stop(set(range(world))) if rank == 0 else None

    def allmax(x):
        if world == 1:
            return float(x)
        t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def allsum(x):
        if world == 1:
            return float(x)
        t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    phase_avg = {k: allmax(sum(p[i] for p in phases) / len(phases))
                 for i, k in enumerate(["pack", "score", "frontier", "merge"])}
    # per-rank phase breakdown: where a missed scaling target goes
    mine = [sum(p[i] for p in phases) / len(phases) for i in range(4)] + [sum(step_ms) / len(step_ms)]
    if world > 1:
        t = torch.tensor(mine, dtype=torch.float64, device=dev)
        allt = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(allt, t)
        per_rank = [[round(float(x), 3) for x in a.tolist()] for a in allt]
    else:
        per_rank = [[round(x, 3) for x in mine]]
    total_ms = allmax(sum(step_ms))
    ms_per_step = total_ms / args.steps
    n_cand = f.n_candidates
    value = n_cand * args.steps / (total_ms / 1000.0)
    # roofline of the dominant kernel (score): algorithmic int ops per launch / its duration
    kern_avg = sum(kern_ms) / len(kern_ms)
    kern_max = allmax(kern_avg)
    # W = 4 algorithmic int ops per K = 2, 3 candidate (add, compare, max,
    # fold) and W = 2 per K = 1 candidate (compare, fold)
    rows_l = pp.partition_rows([m.n_layers for m in w.models], w.n_classes, w.n_batches, 3, rank, world)
    k1_local = sum(w.n_classes * w.n_batches for m in range(len(w.models)) if rows_l[m, 0] == 0 < rows_l[m, 1])
    ops_local = 4 * f.n_candidates_local - 2 * k1_local
    achieved_local = ops_local / (kern_avg / 1000.0)
    peaks = _peaks()
    f_clk = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    peak_ops = SM_COUNT * ISSUE_LANES_PER_CLK_PER_SM * f_clk
    achieved = allsum(achieved_local) / world  # per-GPU average of per-launch rates
    # a stricter floor: one compare per candidate + 3 more ops per feasible one
    min_achieved = allsum((f.n_candidates_local + 3 * f.n_feasible_local) / (kern_avg / 1000.0)) / world
    # Work-based roofline (the integer-issue ceiling): the score phase's executed
    # warp-instructions per step (ncu, profiles/r2_score_ncu.json, this build, config 5 at
    # N = 1; deterministic for the workload) x 32 lanes / the live score-phase time.
    # At N > 1 the ranks split the same work (first-cut-row shards): the per-GPU figure
    # takes 1/N of the N = 1 count over the slowest rank's score time (an approximation:
    # the count is not re-measured per rank).
    prof = score_profile(args.config) if (not args.models and args.margin is None) else None
    traffic = issue = None
    if prof is not None:
        traffic = prof["total"]["dram_bytes"] / world
        issue = prof["total"]["inst_executed"] / world * 32 / (kern_max / 1000.0)
    launches_tot = int(allsum(launches))

    # ---- e2e: through the public API with HOST buffers, H2D + D2H inside the timed region ----
    e2e = None
    if not args.no_e2e:
        rows = pp.partition_rows([m.n_layers for m in w.models], w.n_classes, w.n_batches, 3, rank, world)
        h2d = sum(int(lat_h[m].nbytes + S_h[m].nbytes) for m in range(len(w.models)) if rows[m, 1] > rows[m, 0])
        e2e_steps = args.e2e_steps or args.steps
        # the result is replicated on every rank's device; one host (rank 0) reads it
        host_copy = rank == 0
        pp.update_profiles_async(ctx, lat_h, S_h)
        g = step(copy=host_copy)  # warm the host-copy path
        barrier()
        e_ms, d2h = [], 0
        for _ in range(e2e_steps):
            with torch.cuda.stream(stream):
                flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            pp.update_profiles_async(ctx, lat_h, S_h)  # uploaded by enumerate, overlapped with scoring
            g = step(copy=host_copy)
            e1.record(stream)
            e1.synchronize()
            e_ms.append(e0.elapsed_time(e1))
            d2h = (g.n_points * 32 + (g.n_segments + 1) * 8) if host_copy else 0
        barrier()
        e_tot = allmax(sum(e_ms))
        e2e = {"value": g.n_candidates * e2e_steps / (e_tot / 1000.0), "unit": UNIT,
               "h2d_bytes_per_step": int(allsum(h2d)), "d2h_bytes_per_step": int(allsum(d2h)),
               "ms_per_step": e_tot / e2e_steps,
               "path": "ppipe_update_profiles_async (pinned host lat/S) + ppipe_enumerate (uploads the profiles "
                       "in 7 chunks, each packed (with validation) and scored as it lands, overlapping the H2D) + "
                       "ppipe_pareto(copy_to_host) into a page-locked buffer read zero-copy (rank 0; the merged "
                       "frontier is replicated on every rank's device)"}

    # ---- SLO sweep from the last enumeration: frontier_at
    # truncates every segment to a lower latency target without re-enumerating ----
    sweep = None
    if not args.no_sweep:
        scales = [0.9, 0.8, 0.7, 0.6, 0.5, 0.4, 0.3, 0.2, 0.1]
        pp.frontier_at(ctx, w.slo_us, w.margin_permille, copy_to_host=False)  # warm (buffer allocation)
        barrier()
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        pts = [pp.frontier_at(ctx, (w.slo_us * sc).astype(np.uint32), w.margin_permille, copy_to_host=False).n_points
               for sc in scales]
        s1.record(stream)
        s1.synchronize()
        sweep = {"slo_scales": scales, "ms_per_target": s0.elapsed_time(s1) / len(scales),
                 "frontier_points": pts, "base": "the timed enumeration's frontier (SLO scale 1.0)",
                 "vs": "re-enumerating costs ms_per_step per target"}
    pp.free(ctx)
    # ---- greedy pre-partitioning (§5.2) of this workload's
    # layer-level models into 10 blocks, through the C ABI from pinned host buffers ----
    prepart = None
    if rank == 0 and not args.no_sweep:
        nblk = min(10, min(m.n_layers for m in w.models))
        pp.prepartition(lat_h, S_h, nblk, 1 if w.n_classes > 1 else 0, 0)  # warm
        t0 = time.perf_counter()
        bnd, _, _ = pp.prepartition(lat_h, S_h, nblk, 1 if w.n_classes > 1 else 0, 0)
        prepart = {"models": len(lat_h), "n_blocks": nblk, "ms": (time.perf_counter() - t0) * 1e3,
                   "ref": "class 1, batch index 0", "timing": "host wall clock around ppipe_prepartition "
                   "(H2D of the layer profiles, two kernels, D2H of bounds and block profiles)"}
    # ---- F2, the MILP-lossless frontier, on config 4: one blocking
    # ppipe_pareto_f2 per rep (pack, enumerate, strict-dominance queries, tie runs, sort) ----
    from workloads import CONFIG_NAMES, config4
    f2 = None
    if rank == 0 and not args.no_f2:
        w4 = config4()
        c4 = pp.load_workload(w4, device=local_rank)
        try:
            pp.pareto_f2(c4, w4.kmax, w4.slo_us, w4.margin_permille, copy_to_host=False)  # warm
            reps, dev_ms, wall = 3, [], []
            for _ in range(reps):
                t0 = time.perf_counter()
                r4 = pp.pareto_f2(c4, w4.kmax, w4.slo_us, w4.margin_permille, copy_to_host=False)
                wall.append((time.perf_counter() - t0) * 1e3)
                dev_ms.append(sum(c4.phase_ms()))
            f2 = {"workload": "config 4: " + CONFIG_NAMES[4], "candidates": r4.n_candidates,
                  "feasible": r4.n_feasible, "strict_survivors": r4.n_survivors, "points": r4.n_points,
                  "device_ms": statistics.median(dev_ms), "wall_ms": statistics.median(wall),
                  "candidates_per_s": r4.n_candidates / (statistics.median(wall) / 1e3),
                  "launches": c4.launch_count(),
                  "timing": "median of 3 blocking ppipe_pareto_f2 calls, inputs resident; device_ms = sum of "
                            "the CUDA-event phases (pack, enumerate+queries, ties+sort), wall_ms = host clock"}
        finally:
            pp.free(c4)
    # ---- per-stage batch sizes (App. A.1): every partition at its own
    # batch, B^K times the candidates; on the block-level 18-CNN suite (config 3) and config 4 ----
    pbm = None
    if rank == 0 and not args.no_pb:
        from workloads import config3
        pbm = {}
        for name, wk, reps in (("config 3", config3(), 5), ("config 4", config4(), 2)):
            cx = pp.load_workload(wk, device=local_rank)
            try:
                pp.pareto_pb(cx, wk.kmax, wk.slo_us, wk.margin_permille, copy_to_host=False)  # warm
                dev_ms, wall = [], []
                for _ in range(reps):
                    t0 = time.perf_counter()
                    rp = pp.pareto_pb(cx, wk.kmax, wk.slo_us, wk.margin_permille, copy_to_host=False)
                    wall.append((time.perf_counter() - t0) * 1e3)
                    dev_ms.append(sum(cx.phase_ms()))
                pbm[name] = {"candidates": rp.n_candidates, "feasible": rp.n_feasible, "survivors": rp.n_survivors,
                             "points": rp.n_points, "device_ms": statistics.median(dev_ms),
                             "wall_ms": statistics.median(wall),
                             "candidates_per_s": rp.n_candidates / (statistics.median(wall) / 1e3),
                             "launches": cx.launch_count()}
            finally:
                pp.free(cx)
        pbm["timing"] = ("median of blocking ppipe_pareto_pb calls, inputs resident; candidates = sum_m sum_K "
                         "C(M-1,K-1) C^K B^K, decided per (c2, b3) pair by a sorted feasible-b1 prefix")
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.config)
        g5 = os.path.join(ROOT, "tests", "golden", "config5_oracle.json")
        if args.config == 5 and os.path.exists(g5):  # the whole config 5 on the oracle (scripts/golden_config5.py)
            try:
                gj = json.load(open(g5))
                cpu["config5_in_full"] = {"oracle_sec": gj["total"]["oracle_sec"], "threads": gj["threads"],
                                          "host_cores": gj["host_cores"],
                                          "candidates_per_s": gj["total"]["n_cand"] / gj["total"]["oracle_sec"],
                                          "source": "tests/golden/config5_oracle.json (build host, not this box)"}
            except Exception:
                pass
    per_cfg = None
    if world == 1 and not args.no_per_config and args.config == 5 and not args.models:
        per_cfg = per_config_block(pp, local_rank, with_oracle=not args.no_cpu_baseline)
    from workloads import CONFIG_NAMES
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "int32", "data": "synthetic (seeded; recipe in DESIGN.md §3)",
        "config": {"workload": f"config {args.config}: {CONFIG_NAMES[args.config]}",
                   "candidates_per_step": n_cand, "feasible_per_step": f.n_feasible,
                   "frontier_points": f.n_points, "segments": f.n_segments, "survivors_rank0": f.n_survivors,
                   "l2": "inputs > L2 (P, Y tables ~1.1 GB at N=1) and a 256 MiB L2 flush between timed steps",
                   "parallelism": f"dp{world}: first-cut-row shards + NCCL all-gather frontier merge"
                   if world > 1 else "dp1"},
        "roofline": {"bound": "alu", "achieved": (issue if issue is not None else achieved) / 1e12,
                     "peak": peak_ops / 1e12, "unit": "Tops/s",
                     "frac": (issue if issue is not None else achieved) / peak_ops, "traffic": traffic,
                     "kernel": "score phase (score3a + gfold_prefix + score3b + score12), one step",
                     "kernel_ms": kern_max,
                     "achieved_basis": ("executed warp-instructions of the score kernels per step x 32 lanes / the live "
                                        "score-phase time; instruction and DRAM counts from ncu --set full of this build "
                                        f"({prof['source']})" + (f"; per GPU: 1/{world} of the N = 1 count over the slowest "
                                                                 "rank's score time" if world > 1 else "")
                                        if prof is not None else
                                        "no ncu profile for this configuration: W-model ops (below) instead"),
                     "issue_frac": (issue / peak_ops) if issue is not None else None,
                     "per_kernel_ncu": prof["kernels"] if prof is not None else None,
                     "w_model": {"ops_per_candidate": "SURVEY.md §8(d) W: 4 int32 ops per K=2,3 candidate, 2 per K=1",
                                 "achieved": achieved / 1e12, "frac": achieved / peak_ops,
                                 "note": "effective ops/candidate: above 1 because the 16-bit prefilter decides two "
                                         "candidates per lane-op and the tile bounds decide whole tiles with one "
                                         "compare, so this does not measure executed work",
                                 "frac_one_cmp_plus_3_per_feasible": min_achieved / peak_ops},
                     "peak_basis": f"{SM_COUNT} SMs x {ISSUE_LANES_PER_CLK_PER_SM} int lane-ops/clk (issue) x "
                                   f"{f_clk / 1e6:.0f} MHz (sm_max_mhz, MEASURED_PEAKS.json)"},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches_tot,
        "clocks": clocks,
        "phase_ms": phase_avg,
        "phase_ms_per_rank": {"columns": ["pack", "score", "frontier", "merge", "step"], "ranks": per_rank,
                              "note": "merge includes waiting for the slowest rank at the first all-gather"},
        "slo_sweep": sweep,
        "prepartition": prepart,
        "f2": f2,
        "per_stage_batch": pbm,
        "per_config": per_cfg,
    }
    emit_line(line)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
