"""Multi-rank paths.

* CPU (gloo, world_size 2): the host-side row partition and the decomposability
  of the frontier -- each rank computes the oracle frontier of its rows, the
  local frontiers are all-gathered over gloo and reduced once more; the result
  must equal the single-process oracle.
* GPU (>= 2 devices): the library's own NCCL merge under torchrun
  (scripts/mgpu_check.py), byte-identical to the single-GPU run and the oracle.
"""
from __future__ import annotations

import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from tests.conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, cfg, q):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2507_18748_b200.build import build
        build()
        import paper_2507_18748_b200 as pp
        from oracle import run_oracle
        from tests.helpers import reduce_union
        from workloads import make_config
        w = make_config(cfg)
        rows = pp.partition_rows([m.n_layers for m in w.models], w.n_classes, w.n_batches, 3, rank, world)
        parts = []
        n_cand = 0
        for m in range(len(w.models)):
            lo, hi = int(rows[m, 0]), int(rows[m, 1])
            if hi > lo:
                o = run_oracle(w, model_lo=m, model_hi=m + 1, row_lo=lo, row_hi=hi, threads=2)
                pts = o.points.copy()
                pts["model"] = m
                parts.append(pts)
                n_cand += o.n_candidates
        local = np.concatenate(parts) if parts else np.zeros(0, dtype=parts[0].dtype if parts else None)
        gathered = [None] * world
        dist.all_gather_object(gathered, (local.tobytes(), n_cand))
        if rank == 0:
            from oracle import POINT_DTYPE
            union = np.concatenate([np.frombuffer(b, dtype=POINT_DTYPE) for b, _ in gathered])
            merged = reduce_union(union)
            full = run_oracle(w, threads=2)
            same = np.array_equal(merged.view(np.uint8), full.points.view(np.uint8))
            q.put((same, sum(c for _, c in gathered), full.n_candidates))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg", [2, 3])
def test_gloo_two_rank_partition_and_merge(oracle_built, cfg):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, cfg, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    assert all(p.exitcode == 0 for p in procs)
    same, n_sum, n_full = q.get(timeout=5)
    assert n_sum == n_full
    assert same


def _gloo_f2_worker(rank, world, port, cfg, q):
    """F2 placement: the rank holding a model's row 0 (its K = 1 row) owns the whole model;
    the rank-ordered concatenation of owned frontiers is the global F2 frontier."""
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2507_18748_b200.build import build
        build()
        import paper_2507_18748_b200 as pp
        from oracle import POINT_DTYPE, run_oracle
        from workloads import make_config
        w = make_config(cfg)
        rows = pp.partition_rows([m.n_layers for m in w.models], w.n_classes, w.n_batches, 3, rank, world)
        own = [m for m in range(len(w.models)) if int(rows[m, 0]) == 0 and int(rows[m, 1]) > 0]
        parts = [run_oracle(w, model_lo=m, model_hi=m + 1, threads=2, frontier=2).points for m in own]
        local = np.concatenate(parts) if parts else np.zeros(0, dtype=POINT_DTYPE)
        gathered = [None] * world
        dist.all_gather_object(gathered, (local.tobytes(), own))
        if rank == 0:
            owners = sorted(m for _, o in gathered for m in o)
            union = np.concatenate([np.frombuffer(b, dtype=POINT_DTYPE) for b, _ in gathered])
            full = run_oracle(w, threads=2, frontier=2)
            q.put((owners == list(range(len(w.models))),
                   np.array_equal(union.view(np.uint8), full.points.view(np.uint8))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg", [3])
def test_gloo_two_rank_f2_owned_models(oracle_built, cfg):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_f2_worker, args=(r, 2, port, cfg, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    assert all(p.exitcode == 0 for p in procs)
    each_model_once, same = q.get(timeout=5)
    assert each_model_once and same


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,extra", [(3, ["--oracle"]), (5, ["--models", "24"]),
                                       (4, []),  # one model shared by every rank
                                       (1, ["--oracle"]),  # tiny: some ranks hold no rows
                                       (3, ["--oracle", "--vgpu", "1,2,4,3", "--async-upload"]),
                                       (3, ["--oracle", "--f2"]),  # F2: owned models + all-gather
                                       (5, ["--models", "6", "--f2"]),
                                       (3, ["--oracle", "--pb"])])  # per-stage batch sizes
def test_nccl_two_rank_merge(cfg, extra):
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    n = min(torch.cuda.device_count(), 4)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "scripts", "mgpu_check.py"), "--config", str(cfg), *extra]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "OK" in r.stdout
