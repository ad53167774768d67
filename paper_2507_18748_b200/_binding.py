"""Thin ctypes binding of libppipe_b200.so (include/ppipe.h).

Argument marshalling only: every step of the hot path runs in the library's
CUDA kernels. Same names as the C ABI: load_profiles, enumerate, pareto, free.
There is no CPU fallback: if the library is missing or no sm_100 device is
usable, calls raise PPipeError.
"""
from __future__ import annotations

import ctypes as ct
import os
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# PPIPE_LIB: load another in-tree build of the same sources (tuning experiments, scripts/variants.py)
LIB_PATH = os.environ.get("PPIPE_LIB") or os.path.join(_PKG, "libppipe_b200.so")

PPIPE_OK, PPIPE_EINVAL, PPIPE_ERANGE, PPIPE_ENOMEM, PPIPE_ECUDA, PPIPE_ENCCL, PPIPE_ESTATE = 0, -1, -2, -3, -4, -5, -6
_CODES = {-1: "EINVAL", -2: "ERANGE", -3: "ENOMEM", -4: "ECUDA", -5: "ENCCL", -6: "ESTATE"}

# ppipe_point, 32 bytes (include/ppipe.h)
POINT_DTYPE = np.dtype([
    ("model", "<u4"), ("cut", "<u2", (2,)), ("K", "u1"), ("cls", "u1", (3,)),
    ("batch", "<u2"), ("reserved", "<u2"), ("e2e_us", "<u4"), ("stage_us", "<u4", (3,)),
])
assert POINT_DTYPE.itemsize == 32
# ppipe_point_pb, 32 bytes: per-stage batch INDICES instead of one batch value
POINT_PB_DTYPE = np.dtype([
    ("model", "<u4"), ("cut", "<u2", (2,)), ("K", "u1"), ("cls", "u1", (3,)), ("bidx", "u1", (3,)),
    ("reserved", "u1"), ("e2e_us", "<u4"), ("stage_us", "<u4", (3,)),
])
assert POINT_PB_DTYPE.itemsize == 32


class PPipeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_CODES.get(code, code)}: {msg}")
        self.code = code


class _Model(ct.Structure):
    _fields_ = [("n_layers", ct.c_uint32), ("lat_us", ct.POINTER(ct.c_uint32)),
                ("act_bytes", ct.POINTER(ct.c_uint64))]


class _Dist(ct.Structure):
    _fields_ = [("rank", ct.c_int32), ("world", ct.c_int32), ("device", ct.c_int32), ("nccl_id", ct.c_void_p)]


class _EnumParams(ct.Structure):
    _fields_ = [("max_partitions", ct.c_uint32), ("slo_us", ct.POINTER(ct.c_uint32)),
                ("margin_permille", ct.c_uint32)]


class _Frontier(ct.Structure):
    _fields_ = [("n_candidates", ct.c_uint64), ("n_feasible", ct.c_uint64), ("n_points", ct.c_uint64),
                ("n_segments", ct.c_uint64), ("points", ct.c_void_p), ("seg_offsets", ct.POINTER(ct.c_uint64)),
                ("d_points", ct.c_void_p), ("d_seg_offsets", ct.c_void_p), ("n_survivors", ct.c_uint64),
                ("n_candidates_local", ct.c_uint64), ("n_feasible_local", ct.c_uint64)]


class _FrontierPB(ct.Structure):
    _fields_ = [("n_candidates", ct.c_uint64), ("n_feasible", ct.c_uint64), ("n_points", ct.c_uint64),
                ("n_segments", ct.c_uint64), ("points", ct.c_void_p), ("seg_offsets", ct.POINTER(ct.c_uint64)),
                ("d_points", ct.c_void_p), ("d_seg_offsets", ct.c_void_p), ("n_survivors", ct.c_uint64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise PPipeError(PPIPE_ECUDA, f"{LIB_PATH} is missing: run __graft_entry__.build() "
                                          "(there is no CPU fallback)")
        L = ct.CDLL(LIB_PATH, mode=ct.RTLD_GLOBAL)
        L.ppipe_load_profiles.restype = ct.c_int
        L.ppipe_load_profiles.argtypes = [ct.POINTER(ct.c_void_p), ct.c_uint32, ct.POINTER(_Model), ct.c_uint32,
                                          ct.c_uint32, ct.POINTER(ct.c_uint32), ct.POINTER(ct.c_uint32),
                                          ct.POINTER(_Dist)]
        L.ppipe_update_profiles.restype = ct.c_int
        L.ppipe_update_profiles.argtypes = [ct.c_void_p, ct.c_uint32, ct.POINTER(_Model)]
        L.ppipe_enumerate.restype = ct.c_int
        L.ppipe_enumerate.argtypes = [ct.c_void_p, ct.POINTER(_EnumParams)]
        L.ppipe_pareto.restype = ct.c_int
        L.ppipe_pareto.argtypes = [ct.c_void_p, ct.c_int, ct.POINTER(_Frontier)]
        L.ppipe_prepartition.restype = ct.c_int
        L.ppipe_prepartition.argtypes = [ct.c_uint32, ct.POINTER(_Model), ct.c_uint32, ct.c_uint32, ct.c_uint32,
                                         ct.c_uint32, ct.c_uint32, ct.c_int32, ct.POINTER(ct.c_uint32),
                                         ct.POINTER(ct.c_uint32), ct.POINTER(ct.c_uint64)]
        L.ppipe_update_profiles_async.restype = ct.c_int
        L.ppipe_update_profiles_async.argtypes = [ct.c_void_p, ct.c_uint32, ct.POINTER(_Model)]
        L.ppipe_set_vgpu.restype = ct.c_int
        L.ppipe_set_vgpu.argtypes = [ct.c_void_p, ct.POINTER(ct.c_uint8)]
        L.ppipe_pareto_pb.restype = ct.c_int
        L.ppipe_pareto_pb.argtypes = [ct.c_void_p, ct.POINTER(_EnumParams), ct.c_int, ct.POINTER(_FrontierPB)]
        L.ppipe_pareto_f2.restype = ct.c_int
        L.ppipe_pareto_f2.argtypes = [ct.c_void_p, ct.POINTER(_EnumParams), ct.c_int, ct.POINTER(_Frontier)]
        L.ppipe_frontier_at.restype = ct.c_int
        L.ppipe_frontier_at.argtypes = [ct.c_void_p, ct.POINTER(ct.c_uint32), ct.c_uint32, ct.c_int,
                                        ct.POINTER(_Frontier)]
        L.ppipe_merge_shards.restype = ct.c_int
        L.ppipe_merge_shards.argtypes = [ct.POINTER(ct.c_void_p), ct.c_int, ct.c_int, ct.POINTER(_Frontier)]
        L.ppipe_free.restype = None
        L.ppipe_free.argtypes = [ct.c_void_p]
        L.ppipe_last_error.restype = ct.c_char_p
        L.ppipe_last_error.argtypes = [ct.c_void_p]
        L.ppipe_nccl_unique_id.restype = ct.c_int
        L.ppipe_nccl_unique_id.argtypes = [ct.c_void_p]
        L.ppipe_stream.restype = ct.c_void_p
        L.ppipe_stream.argtypes = [ct.c_void_p]
        L.ppipe_phase_ms.restype = ct.c_int
        L.ppipe_phase_ms.argtypes = [ct.c_void_p, ct.POINTER(ct.c_float)]
        L.ppipe_launch_count.restype = ct.c_uint64
        L.ppipe_launch_count.argtypes = [ct.c_void_p]
        L.ppipe_partition_rows.restype = ct.c_int
        L.ppipe_partition_rows.argtypes = [ct.c_uint32, ct.POINTER(ct.c_uint32), ct.c_uint32, ct.c_uint32,
                                           ct.c_uint32, ct.c_int32, ct.c_int32, ct.POINTER(ct.c_uint32)]
        _lib = L
    return _lib


def _check(rc: int, ctx=None):
    if rc != PPIPE_OK:
        msg = lib().ppipe_last_error(ctx)
        raise PPipeError(rc, msg.decode() if msg else "")


def _u32p(a):
    return a.ctypes.data_as(ct.POINTER(ct.c_uint32))


class Context:
    """Owns a ppipe_ctx* plus the host arrays it was built from."""

    def __init__(self, handle, n_models, n_classes=None, n_batches=None):
        self.handle = handle
        self.n_models = n_models
        self.n_classes = n_classes
        self.n_batches = n_batches

    @property
    def stream(self) -> int:
        return int(lib().ppipe_stream(self.handle) or 0)

    def phase_ms(self):
        out = (ct.c_float * 4)()
        _check(lib().ppipe_phase_ms(self.handle, out), self.handle)
        return [float(x) for x in out]

    def launch_count(self) -> int:
        return int(lib().ppipe_launch_count(self.handle))


def nccl_unique_id() -> bytes:
    buf = ct.create_string_buffer(128)
    _check(lib().ppipe_nccl_unique_id(buf))
    return buf.raw


# ppipe_model as a numpy record (u32 n_layers, 4 bytes padding, two pointers): the array
# of descriptors is built without one ctypes object per model
_MODEL_REC = np.dtype([("n_layers", "<u4"), ("pad", "<u4"), ("lat_us", "<u8"), ("act_bytes", "<u8")])
assert _MODEL_REC.itemsize == ct.sizeof(_Model)


def _models_array(lat_us, act_bytes, n_classes=None, n_batches=None):
    n = len(lat_us)
    if len(act_bytes) != n:
        raise PPipeError(PPIPE_EINVAL, f"{n} latency arrays but {len(act_bytes)} act_bytes arrays")
    rec = np.zeros(max(n, 1), dtype=_MODEL_REC)
    keep = [rec]
    nl, pl, ps = [0] * n, [0] * n, [0] * n
    for i in range(n):
        lat, S = lat_us[i], act_bytes[i]
        if type(lat) is not np.ndarray or lat.dtype != np.uint32 or not lat.flags.c_contiguous:
            lat = np.ascontiguousarray(lat, dtype=np.uint32)
            keep.append(lat)
        if type(S) is not np.ndarray or S.dtype != np.uint64 or not S.flags.c_contiguous:
            S = np.ascontiguousarray(S, dtype=np.uint64)
            keep.append(S)
        sh = lat.shape
        if len(sh) != 3 or (n_classes is not None and sh[0] != n_classes) or \
                (n_batches is not None and sh[2] != n_batches) or S.shape != (sh[1],):
            raise PPipeError(PPIPE_EINVAL, f"model {i}: lat_us must be [n_classes][n_layers][n_batches] and "
                                           f"act_bytes [n_layers]; got {sh} and {S.shape}")
        nl[i] = sh[1]
        pl[i] = lat.__array_interface__["data"][0]
        ps[i] = S.__array_interface__["data"][0]
    if n:
        rec["n_layers"][:n] = nl
        rec["lat_us"][:n] = pl
        rec["act_bytes"][:n] = ps
    keep += [lat_us, act_bytes]
    return ct.cast(rec.ctypes.data, ct.POINTER(_Model)), keep


def update_profiles(ctx: Context, lat_us: Sequence[np.ndarray], act_bytes: Sequence[np.ndarray]) -> None:
    models, keep = _models_array(lat_us, act_bytes, ctx.n_classes, ctx.n_batches)
    _check(lib().ppipe_update_profiles(ctx.handle, len(lat_us), models), ctx.handle)
    del keep


def update_profiles_async(ctx: Context, lat_us: Sequence[np.ndarray], act_bytes: Sequence[np.ndarray]) -> None:
    """include/ppipe.h ppipe_update_profiles_async: the next enumerate() uploads the
    values in chunks overlapped with scoring. The arrays must stay alive and unchanged
    until the next pareto() returns (the context keeps references until then)."""
    # The descriptor array of the same array objects as the last call is reused (a serving
    # loop re-uploads the same pinned buffers with new contents; building the 1,000
    # descriptors costs ~2 ms of Python). An ndarray's data pointer cannot move while we
    # hold a reference to it; its shape and dtype are re-checked.
    last = getattr(ctx, "_desc_cache", None)
    if last is not None and len(last[0]) == len(lat_us) and len(last[1]) == len(act_bytes) and \
            all(a is b and a.shape == sh and a.dtype == np.uint32 for a, b, sh in zip(lat_us, last[0], last[4])) and \
            all(a is b and a.shape == sh and a.dtype == np.uint64 for a, b, sh in zip(act_bytes, last[1], last[5])):
        models, keep = last[2], last[3]
    else:
        models, keep = _models_array(lat_us, act_bytes, ctx.n_classes, ctx.n_batches)
        # (cached only when no input needed a conversion: keep = [descriptors, lat_us, act_bytes])
        ctx._desc_cache = (tuple(lat_us), tuple(act_bytes), models, keep, tuple(a.shape for a in lat_us),
                           tuple(a.shape for a in act_bytes)) if len(keep) == 3 else None
    _check(lib().ppipe_update_profiles_async(ctx.handle, len(lat_us), models), ctx.handle)
    ctx._pending = keep  # keep the buffers alive for the deferred copy


def load_profiles(lat_us: Sequence[np.ndarray], act_bytes: Sequence[np.ndarray], n_classes: int,
                  batches: np.ndarray, bw_bits_per_us: np.ndarray, rank: int = 0, world: int = 1,
                  device: int = -1, nccl_id: Optional[bytes] = None) -> Context:
    n = len(lat_us)
    b = np.ascontiguousarray(batches, dtype=np.uint32)
    models, keep = _models_array(lat_us, act_bytes, n_classes, len(b))
    bw = np.ascontiguousarray(bw_bits_per_us, dtype=np.uint32).reshape(-1)
    idbuf = ct.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
    dist = _Dist(rank, world, device, ct.cast(idbuf, ct.c_void_p) if idbuf is not None else None)
    h = ct.c_void_p()
    rc = lib().ppipe_load_profiles(ct.byref(h), n, models, n_classes, len(b), _u32p(b), _u32p(bw), ct.byref(dist))
    _check(rc, None)
    del keep
    return Context(h, n, int(n_classes), len(b))


def load_workload(w, rank: int = 0, world: int = 1, device: int = -1, nccl_id: Optional[bytes] = None) -> Context:
    """Convenience: load a workloads.Workload."""
    return load_profiles([m.lat_us for m in w.models], [m.act_bytes for m in w.models], w.n_classes,
                         w.batches, w.bw, rank, world, device, nccl_id)


def enumerate(ctx: Context, max_partitions: int, slo_us: np.ndarray, margin_permille: int) -> None:  # noqa: A001
    slo = np.ascontiguousarray(slo_us, dtype=np.uint32)
    if slo.shape[0] != ctx.n_models:
        raise PPipeError(PPIPE_EINVAL, f"slo_us has {slo.shape[0]} entries for {ctx.n_models} models")
    p = _EnumParams(max_partitions, _u32p(slo), margin_permille)
    _check(lib().ppipe_enumerate(ctx.handle, ct.byref(p)), ctx.handle)


@dataclass
class Frontier:
    n_candidates: int
    n_feasible: int
    n_points: int
    n_segments: int
    n_survivors: int
    points: Optional[np.ndarray]       # POINT_DTYPE (host), canonical order
    seg_offsets: Optional[np.ndarray]  # uint64 [n_segments + 1]
    d_points: int                      # device pointer
    d_seg_offsets: int
    n_candidates_local: int = 0
    n_feasible_local: int = 0


def _frontier_from(f, copy_to_host: bool, zero_copy: bool, dtype=POINT_DTYPE) -> Frontier:
    pts = seg = None
    if copy_to_host:
        n = int(f.n_points)
        if n:
            buf = (ct.c_char * (32 * n)).from_address(f.points)
            pts = np.frombuffer(buf, dtype=dtype)
            if not zero_copy:
                pts = pts.copy()
        else:
            pts = np.zeros(0, dtype=dtype)
        seg = np.ctypeslib.as_array(f.seg_offsets, shape=(int(f.n_segments) + 1,))
        if not zero_copy:
            seg = seg.copy()
    return Frontier(int(f.n_candidates), int(f.n_feasible), int(f.n_points), int(f.n_segments),
                    int(f.n_survivors), pts, seg, int(f.d_points or 0), int(f.d_seg_offsets or 0),
                    int(getattr(f, "n_candidates_local", 0)), int(getattr(f, "n_feasible_local", 0)))


def pareto(ctx: Context, copy_to_host: bool = True, zero_copy: bool = False) -> Frontier:
    """Run the frontier pass. copy_to_host: also return host arrays. zero_copy: those
    arrays are views of the context's page-locked result buffer (no host memcpy),
    valid only until the next pareto() / frontier_at() / free() on this context."""
    f = _Frontier()
    _check(lib().ppipe_pareto(ctx.handle, 1 if copy_to_host else 0, ct.byref(f)), ctx.handle)
    return _frontier_from(f, copy_to_host, zero_copy)


def merge_shards(ctxs: Sequence[Context], copy_to_host: bool = True, zero_copy: bool = False) -> Frontier:
    """Merge the local frontiers of shard-mode contexts (rank r of len(ctxs), no NCCL id,
    one GPU) with the library's multi-GPU merge (include/ppipe.h ppipe_merge_shards).
    The result is owned by ctxs[0]."""
    arr = (ct.c_void_p * len(ctxs))(*[c.handle for c in ctxs])
    f = _Frontier()
    _check(lib().ppipe_merge_shards(arr, len(ctxs), 1 if copy_to_host else 0, ct.byref(f)), ctxs[0].handle)
    return _frontier_from(f, copy_to_host, zero_copy)


def pareto_f2(ctx: Context, max_partitions: int, slo_us: np.ndarray, margin_permille: int,
              copy_to_host: bool = True, zero_copy: bool = False) -> Frontier:
    """F2, the MILP-lossless per-stage throughput frontier (include/ppipe.h
    ppipe_pareto_f2): pack, enumerate and reduce in one blocking call; points in
    (segment, b, c_1, c_2) order."""
    slo = np.ascontiguousarray(slo_us, dtype=np.uint32)
    if slo.shape[0] != ctx.n_models:
        raise PPipeError(PPIPE_EINVAL, f"slo_us has {slo.shape[0]} entries for {ctx.n_models} models")
    p = _EnumParams(max_partitions, _u32p(slo), margin_permille)
    f = _Frontier()
    _check(lib().ppipe_pareto_f2(ctx.handle, ct.byref(p), 1 if copy_to_host else 0, ct.byref(f)), ctx.handle)
    return _frontier_from(f, copy_to_host, zero_copy)


def pareto_pb(ctx: Context, max_partitions: int, slo_us: np.ndarray, margin_permille: int,
              copy_to_host: bool = True, zero_copy: bool = False) -> Frontier:
    """Per-stage batch sizes (include/ppipe.h ppipe_pareto_pb): every partition at its own
    batch; points are POINT_PB_DTYPE (batch indices per stage), per segment E-ascending."""
    slo = np.ascontiguousarray(slo_us, dtype=np.uint32)
    if slo.shape[0] != ctx.n_models:
        raise PPipeError(PPIPE_EINVAL, f"slo_us has {slo.shape[0]} entries for {ctx.n_models} models")
    p = _EnumParams(max_partitions, _u32p(slo), margin_permille)
    f = _FrontierPB()
    _check(lib().ppipe_pareto_pb(ctx.handle, ct.byref(p), 1 if copy_to_host else 0, ct.byref(f)), ctx.handle)
    return _frontier_from(f, copy_to_host, zero_copy, POINT_PB_DTYPE)


def frontier_at(ctx: Context, slo_us: np.ndarray, margin_permille: int, copy_to_host: bool = True,
                zero_copy: bool = False) -> Frontier:
    """The frontier at lower per-model SLOs, truncated from the last pareto() result
    (include/ppipe.h ppipe_frontier_at; no re-enumeration)."""
    slo = np.ascontiguousarray(slo_us, dtype=np.uint32)
    if slo.shape[0] != ctx.n_models:
        raise ValueError(f"slo_us has {slo.shape[0]} entries, context has {ctx.n_models} models")
    f = _Frontier()
    _check(lib().ppipe_frontier_at(ctx.handle, _u32p(slo), int(margin_permille), 1 if copy_to_host else 0,
                                   ct.byref(f)), ctx.handle)
    return _frontier_from(f, copy_to_host, zero_copy)


def prepartition(lat_us: Sequence[np.ndarray], act_bytes: Sequence[np.ndarray], n_blocks: int, ref_class: int = 0,
                 ref_batch: int = 0, device: int = -1):
    """Greedy equal-runtime pre-partitioning on the GPU (include/ppipe.h ppipe_prepartition).
    Returns (bounds [n_models][n_blocks+1] uint32, block latencies: list of uint32
    [C][n_blocks][B] arrays, block bytes [n_models][n_blocks] uint64)."""
    n = len(lat_us)
    if n == 0:
        return np.zeros((0, n_blocks + 1), np.uint32), [], np.zeros((0, n_blocks), np.uint64)
    C, _, B = np.asarray(lat_us[0]).shape
    models, keep = _models_array(lat_us, act_bytes, C, B)
    N = int(n_blocks)
    bounds = np.zeros((n, N + 1), dtype=np.uint32)
    blat = np.zeros((n, C, N, B), dtype=np.uint32)
    bS = np.zeros((n, N), dtype=np.uint64)
    rc = lib().ppipe_prepartition(n, models, C, B, N, int(ref_class), int(ref_batch), int(device), _u32p(bounds),
                                  _u32p(blat), bS.ctypes.data_as(ct.POINTER(ct.c_uint64)))
    _check(rc, None)
    del keep
    return bounds, [blat[m] for m in range(n)], bS


def set_vgpu(ctx: Context, vgpu: Optional[Sequence[int]]) -> None:
    """Per-class virtual-GPU counts (include/ppipe.h ppipe_set_vgpu); None = all 1."""
    if vgpu is None:
        _check(lib().ppipe_set_vgpu(ctx.handle, None), ctx.handle)
        return
    arr = (ct.c_uint8 * len(vgpu))(*[int(v) for v in vgpu])
    _check(lib().ppipe_set_vgpu(ctx.handle, arr), ctx.handle)


def free(ctx: Context) -> None:
    if ctx is not None and ctx.handle:
        lib().ppipe_free(ctx.handle)
        ctx.handle = None


def partition_rows(n_layers: Sequence[int], n_classes: int, n_batches: int, max_partitions: int, rank: int,
                   world: int) -> np.ndarray:
    Ms = np.ascontiguousarray(n_layers, dtype=np.uint32)
    rows = np.zeros(2 * len(Ms), dtype=np.uint32)
    _check(lib().ppipe_partition_rows(len(Ms), _u32p(Ms), n_classes, n_batches, max_partitions, rank, world,
                                      _u32p(rows)))
    return rows.reshape(-1, 2)


def run(w, rank: int = 0, world: int = 1, device: int = -1, nccl_id: Optional[bytes] = None,
        copy_to_host: bool = True, vgpu: Optional[Sequence[int]] = None, frontier: int = 1) -> Frontier:
    """One full pass: load, (set_vgpu), enumerate, pareto, free. frontier=2: F2 (pareto_f2);
    frontier=3: per-stage batch sizes (pareto_pb)."""
    ctx = load_workload(w, rank, world, device, nccl_id)
    try:
        if vgpu is not None:
            set_vgpu(ctx, vgpu)
        if frontier == 2:
            return pareto_f2(ctx, w.kmax, w.slo_us, w.margin_permille, copy_to_host)
        if frontier == 3:
            return pareto_pb(ctx, w.kmax, w.slo_us, w.margin_permille, copy_to_host)
        enumerate(ctx, w.kmax, w.slo_us, w.margin_permille)
        return pareto(ctx, copy_to_host)
    finally:
        free(ctx)
