"""B200-native PPipe plan enumeration (arXiv 2507.18748): the data-parallel hot
path of PPipe's control plane -- exhaustive enumeration and scoring of
pool-based pipeline plans and their reduction to a per-(model, K, class tuple)
Pareto frontier -- as hand-written sm_100a CUDA kernels behind a C ABI
(include/ppipe.h). See DESIGN.md.
"""
from ._binding import (  # noqa: F401
    POINT_DTYPE,
    POINT_PB_DTYPE,
    Context,
    Frontier,
    PPipeError,
    enumerate,
    free,
    frontier_at,
    load_profiles,
    load_workload,
    merge_shards,
    nccl_unique_id,
    pareto,
    pareto_f2,
    pareto_pb,
    partition_rows,
    prepartition,
    run,
    set_vgpu,
    update_profiles,
    update_profiles_async,
    lib,
    LIB_PATH,
)
