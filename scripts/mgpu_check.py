"""Multi-GPU parity check (run under torchrun, one process per GPU).

Every rank enumerates its first-cut-row shard of the workload and ppipe_pareto
merges the local frontiers with NCCL all-gather + one final frontier pass
(SURVEY.md §8(e)). Rank 0 checks that the merged frontier (replicated on every
rank) is byte-identical to the single-GPU result and, for small configs, to the
CPU oracle. Exit code 0 on success.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29511 scripts/mgpu_check.py --config 3
"""
from __future__ import annotations

import argparse
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--models", type=int, default=None)
    ap.add_argument("--oracle", action="store_true", help="also compare with the CPU oracle (small configs)")
    ap.add_argument("--vgpu", type=str, default=None, help="comma-separated per-class virtual-GPU counts")
    ap.add_argument("--async-upload", action="store_true", help="load scaled values, then update_profiles_async")
    ap.add_argument("--f2", action="store_true", help="F2 frontier (ppipe_pareto_f2): owned models + all-gather")
    ap.add_argument("--pb", action="store_true", help="per-stage batch sizes (ppipe_pareto_pb): owned models")
    args = ap.parse_args()
    kind = 2 if args.f2 else (3 if args.pb else 1)

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2507_18748_b200 as pp
    from workloads import make_config

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    kw = {"n_models": args.models} if (args.models and args.config == 5) else {}
    w = make_config(args.config, **kw)
    t = torch.zeros(128, dtype=torch.uint8, device=dev)
    if rank == 0:
        t.copy_(torch.frombuffer(bytearray(pp.nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(t, 0)
    nid = bytes(t.cpu().numpy().tobytes())
    vgpu = [int(x) for x in args.vgpu.split(",")] if args.vgpu else None
    if args.async_upload:
        scaled = [np.minimum(m.lat_us.astype(np.uint64) * 5 // 4, 1 << 20).astype(np.uint32) for m in w.models]
        ctx = pp.load_profiles(scaled, [m.act_bytes for m in w.models], w.n_classes, w.batches, w.bw, rank=rank,
                               world=world, device=local, nccl_id=nid)
        try:
            if vgpu:
                pp.set_vgpu(ctx, vgpu)
            pp.update_profiles_async(ctx, [m.lat_us for m in w.models], [m.act_bytes for m in w.models])
            pp.enumerate(ctx, w.kmax, w.slo_us, w.margin_permille)
            g = pp.pareto(ctx)
        finally:
            pp.free(ctx)
    else:
        g = pp.run(w, rank=rank, world=world, device=local, nccl_id=nid, vgpu=vgpu, frontier=kind)
    digest = hashlib.sha256(g.points.tobytes() + g.seg_offsets.tobytes()).hexdigest()
    digests = [None] * world
    dist.all_gather_object(digests, (digest, g.n_candidates, g.n_feasible, g.n_points))
    ok = True
    if rank == 0:
        if len(set(digests)) != 1:
            print("ranks disagree:", digests)
            ok = False
        single = pp.run(w, device=local, vgpu=vgpu, frontier=kind)
        if not (np.array_equal(single.points.view(np.uint8), g.points.view(np.uint8))
                and np.array_equal(single.seg_offsets, g.seg_offsets)
                and single.n_candidates == g.n_candidates and single.n_feasible == g.n_feasible):
            print(f"{world}-rank result differs from the single-GPU result "
                  f"({g.n_points} vs {single.n_points} points)")
            ok = False
        if args.oracle:
            from oracle import run_oracle, run_oracle_pb
            o = run_oracle_pb(w) if kind == 3 else run_oracle(w, vgpu=vgpu, frontier=kind)
            if not (np.array_equal(o.points.view(np.uint8), g.points.view(np.uint8))
                    and o.n_candidates == g.n_candidates and o.n_feasible == g.n_feasible):
                print("multi-GPU result differs from the oracle")
                ok = False
        print(f"mgpu_check config {args.config} world {world}: {'OK' if ok else 'FAIL'} "
              f"({g.n_candidates} candidates, {g.n_feasible} feasible, {g.n_points} points, digest {digest[:16]})")
    okt = torch.tensor([1 if ok else 0], device=dev)
    dist.broadcast(okt, 0)
    dist.barrier()
    dist.destroy_process_group()
    return 0 if okt.item() == 1 else 1


if __name__ == "__main__":
    sys.exit(main())
