"""ctypes wrapper around oracle/ppipe_oracle.c (test infrastructure only).

See ppipe_oracle.c's header for the definition it follows (PAPER.md citations)
and tests/test_oracle_pins.py for what pins it.
"""
from __future__ import annotations

import ctypes as ct
import os
import subprocess
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ppipe_oracle.c")
_LIB = os.path.join(_HERE, "libppipe_oracle.so")

# 32-byte point record (field layout documented in DESIGN.md §4); defined here
# independently of the product binding.
POINT_DTYPE = np.dtype([
    ("model", "<u4"), ("cut", "<u2", (2,)), ("K", "u1"), ("cls", "u1", (3,)),
    ("batch", "<u2"), ("reserved", "<u2"), ("e2e_us", "<u4"), ("stage_us", "<u4", (3,)),
])
assert POINT_DTYPE.itemsize == 32
# per-stage batch records (oracle_run_pb): batch INDICES per stage instead of one batch value
POINT_PB_DTYPE = np.dtype([
    ("model", "<u4"), ("cut", "<u2", (2,)), ("K", "u1"), ("cls", "u1", (3,)), ("bidx", "u1", (3,)),
    ("reserved", "u1"), ("e2e_us", "<u4"), ("stage_us", "<u4", (3,)),
])
assert POINT_PB_DTYPE.itemsize == 32


def oracle_lib_path() -> str:
    return _LIB


def build_oracle(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-Wall", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lpthread"])
    return _LIB


class _Model(ct.Structure):
    _fields_ = [("n_layers", ct.c_uint32), ("lat_us", ct.POINTER(ct.c_uint32)),
                ("act_bytes", ct.POINTER(ct.c_uint64))]


class _Result(ct.Structure):
    _fields_ = [("pts", ct.c_void_p), ("n_pts", ct.c_uint64), ("seg_off", ct.POINTER(ct.c_uint64)),
                ("n_seg", ct.c_uint64), ("n_cand", ct.c_uint64), ("n_feas", ct.c_uint64)]


_lib = None


def _load():
    global _lib
    if _lib is None:
        build_oracle()
        lib = ct.CDLL(_LIB)
        lib.oracle_run.restype = ct.c_int
        lib.oracle_run.argtypes = [ct.c_uint32, ct.POINTER(_Model), ct.c_uint32, ct.c_uint32,
                                   ct.POINTER(ct.c_uint32), ct.POINTER(ct.c_uint32), ct.c_uint32,
                                   ct.POINTER(ct.c_uint32), ct.c_uint32, ct.c_uint32, ct.c_uint32,
                                   ct.c_int, ct.POINTER(ct.c_uint8), ct.c_int32, ct.c_int32,
                                   ct.POINTER(ct.POINTER(_Result))]
        lib.oracle_result_free.argtypes = [ct.POINTER(_Result)]
        lib.oracle_set_threads.argtypes = [ct.c_int]
        lib.oracle_set_vgpu.argtypes = [ct.POINTER(ct.c_uint8), ct.c_uint32]
        lib.oracle_set_frontier.argtypes = [ct.c_int]
        lib.oracle_run_pb.restype = ct.c_int
        lib.oracle_run_pb.argtypes = [ct.c_uint32, ct.POINTER(_Model), ct.c_uint32, ct.c_uint32,
                                      ct.POINTER(ct.c_uint32), ct.POINTER(ct.c_uint32), ct.c_uint32,
                                      ct.POINTER(ct.c_uint32), ct.c_uint32, ct.c_uint32, ct.c_uint32,
                                      ct.POINTER(ct.POINTER(_Result))]
        lib.oracle_result_pb_free.argtypes = [ct.POINTER(_Result)]
        lib.oracle_prepartition.restype = ct.c_int
        lib.oracle_prepartition.argtypes = [ct.c_uint32, ct.c_uint32, ct.c_uint32, ct.POINTER(ct.c_uint32),
                                            ct.POINTER(ct.c_uint64), ct.c_uint32, ct.c_uint32, ct.c_uint32,
                                            ct.POINTER(ct.c_uint32), ct.POINTER(ct.c_uint64),
                                            ct.POINTER(ct.c_uint64)]
        _lib = lib
    return _lib


@dataclass
class OracleResult:
    points: np.ndarray  # POINT_DTYPE, canonical order
    seg_offsets: np.ndarray  # uint64 [n_seg + 1]
    n_candidates: int
    n_feasible: int


def _u32p(a: np.ndarray):
    return a.ctypes.data_as(ct.POINTER(ct.c_uint32))


def run_oracle(w, model_lo: int = 0, model_hi: Optional[int] = None, only_K: int = 0,
               only_cls: Optional[Sequence[int]] = None, row_lo: int = 0, row_hi: int = 0,
               threads: int = 0, slo_us: Optional[np.ndarray] = None,
               margin_permille: Optional[int] = None, kmax: Optional[int] = None,
               vgpu: Optional[Sequence[int]] = None, frontier: int = 1) -> OracleResult:
    """Run the oracle on a workloads.Workload (or a sub-range of its models).
    vgpu: per-class virtual-GPU count v_k (theta = min_d v_d b / C_d); None = all 1.
    frontier: 1 = the (E, theta) staircase, 2 = F2, the MILP-lossless per-stage
    throughput frontier (ppipe_oracle.c, f2_beats)."""
    lib = _load()
    lib.oracle_set_threads(int(threads))
    lib.oracle_set_frontier(int(frontier))
    if vgpu is not None:
        varr = (ct.c_uint8 * w.n_classes)(*[int(v) for v in vgpu])
        lib.oracle_set_vgpu(varr, w.n_classes)
    else:
        lib.oracle_set_vgpu(None, 0)
    n = len(w.models)
    model_hi = n if model_hi is None else model_hi
    keep = []
    models = (_Model * max(n, 1))()
    for i, mp in enumerate(w.models):
        lat = np.ascontiguousarray(mp.lat_us, dtype=np.uint32)
        S = np.ascontiguousarray(mp.act_bytes, dtype=np.uint64)
        if lat.ndim != 3 or lat.shape[0] != w.n_classes or lat.shape[2] != w.n_batches or S.shape != (lat.shape[1],):
            raise ValueError(f"model {i}: lat_us {lat.shape} / act_bytes {S.shape} do not match the workload")
        keep += [lat, S]
        models[i].n_layers = lat.shape[1]
        models[i].lat_us = _u32p(lat)
        models[i].act_bytes = S.ctypes.data_as(ct.POINTER(ct.c_uint64))
    batches = np.ascontiguousarray(w.batches, dtype=np.uint32)
    bw = np.ascontiguousarray(w.bw, dtype=np.uint32).reshape(-1)
    slo = np.ascontiguousarray(w.slo_us if slo_us is None else slo_us, dtype=np.uint32)
    cls_arr = None
    if only_cls is not None:
        cls_arr = (ct.c_uint8 * 3)(*(list(only_cls) + [0] * (3 - len(only_cls))))
    out = ct.POINTER(_Result)()
    rc = lib.oracle_run(n, models, w.n_classes, w.n_batches, _u32p(batches), _u32p(bw),
                        w.kmax if kmax is None else kmax, _u32p(slo),
                        w.margin_permille if margin_permille is None else margin_permille,
                        model_lo, model_hi, int(only_K), cls_arr, int(row_lo), int(row_hi), ct.byref(out))
    if rc != 0:
        raise ValueError(f"oracle_run rejected its input (rc={rc})")
    r = out.contents
    npts = int(r.n_pts)
    if npts:
        buf = (ct.c_char * (npts * 32)).from_address(r.pts)
        pts = np.frombuffer(bytes(buf), dtype=POINT_DTYPE).copy()
    else:
        pts = np.zeros(0, dtype=POINT_DTYPE)
    seg = np.ctypeslib.as_array(r.seg_off, shape=(int(r.n_seg) + 1,)).copy()
    res = OracleResult(pts, seg, int(r.n_cand), int(r.n_feas))
    lib.oracle_result_free(out)
    del keep
    return res


def run_oracle_pb(w, model_lo: int = 0, model_hi: Optional[int] = None, threads: int = 0,
                  slo_us: Optional[np.ndarray] = None, kmax: Optional[int] = None) -> OracleResult:
    """Per-stage batch sizes (oracle_run_pb in ppipe_oracle.c): every partition picks its own
    batch; records are POINT_PB_DTYPE (batch indices per stage)."""
    lib = _load()
    lib.oracle_set_threads(int(threads))
    n = len(w.models)
    model_hi = n if model_hi is None else model_hi
    keep = []
    models = (_Model * max(n, 1))()
    for i, mp in enumerate(w.models):
        lat = np.ascontiguousarray(mp.lat_us, dtype=np.uint32)
        S = np.ascontiguousarray(mp.act_bytes, dtype=np.uint64)
        keep += [lat, S]
        models[i].n_layers = lat.shape[1]
        models[i].lat_us = _u32p(lat)
        models[i].act_bytes = S.ctypes.data_as(ct.POINTER(ct.c_uint64))
    batches = np.ascontiguousarray(w.batches, dtype=np.uint32)
    bw = np.ascontiguousarray(w.bw, dtype=np.uint32).reshape(-1)
    slo = np.ascontiguousarray(w.slo_us if slo_us is None else slo_us, dtype=np.uint32)
    out = ct.POINTER(_Result)()
    rc = lib.oracle_run_pb(n, models, w.n_classes, w.n_batches, _u32p(batches), _u32p(bw),
                           w.kmax if kmax is None else kmax, _u32p(slo), w.margin_permille, model_lo, model_hi,
                           ct.byref(out))
    if rc != 0:
        raise ValueError(f"oracle_run_pb rejected its input (rc={rc})")
    r = out.contents
    npts = int(r.n_pts)
    if npts:
        buf = (ct.c_char * (npts * 32)).from_address(r.pts)
        pts = np.frombuffer(bytes(buf), dtype=POINT_PB_DTYPE).copy()
    else:
        pts = np.zeros(0, dtype=POINT_PB_DTYPE)
    seg = np.ctypeslib.as_array(r.seg_off, shape=(int(r.n_seg) + 1,)).copy()
    res = OracleResult(pts, seg, int(r.n_cand), int(r.n_feas))
    lib.oracle_result_pb_free(out)
    del keep
    return res


def prepartition_oracle(lat_us: np.ndarray, act_bytes: np.ndarray, n_blocks: int, ref_class: int, ref_batch: int):
    """Greedy equal-runtime pre-partitioning (oracle_prepartition in ppipe_oracle.c).
    Returns (bounds[N+1] uint32, block_lat[C][N][B] uint64, block_S[N] uint64)."""
    lib = _load()
    lat = np.ascontiguousarray(lat_us, dtype=np.uint32)
    S = np.ascontiguousarray(act_bytes, dtype=np.uint64)
    C, M, B = lat.shape
    if S.shape != (M,):
        raise ValueError("act_bytes must have one entry per layer")
    N = int(n_blocks)
    bounds = np.zeros(max(N, 0) + 1, dtype=np.uint32)
    blat = np.zeros((C, max(N, 1), B), dtype=np.uint64)
    bS = np.zeros(max(N, 1), dtype=np.uint64)
    rc = lib.oracle_prepartition(M, C, B, _u32p(lat), S.ctypes.data_as(ct.POINTER(ct.c_uint64)), N, int(ref_class),
                                 int(ref_batch), _u32p(bounds), blat.ctypes.data_as(ct.POINTER(ct.c_uint64)),
                                 bS.ctypes.data_as(ct.POINTER(ct.c_uint64)))
    if rc != 0:
        raise ValueError(f"oracle_prepartition rejected its input (N={N}, M={M})")
    return bounds, blat, bS
