"""Seeded synthetic PPipe planning workloads (input recipe only).

This package is shared by the CPU oracle tests and the CUDA path. It holds
only input generation (profile tables, feature-map sizes, bandwidth matrix,
SLOs); none of the hot path's arithmetic (stage latency, transfer time, E2E
latency, feasibility, throughput, frontier) lives here. See DESIGN.md
"Input recipe" and SURVEY.md §8(d).

One labelled exception, an INPUT step rather than the method under test:
config 3's block-level models are built by grouping layer-level synthetic
models into N = 10 blocks (generate._prepartition_input_step), the paper's
planning granularity (§5.2). It is a float-target variant
written for input construction only; the product's greedy pre-partitioner
(ppipe_prepartition) and the oracle's (oracle_prepartition) are separate
implementations, checked against each other and their pins in
tests/test_prepartition_{pins,gpu}.py, and neither reads this one.
"""
from .generate import (  # noqa: F401
    Workload,
    ModelProfile,
    CLASS_LIBRARY,
    make_config,
    config1,
    config2,
    config3,
    config4,
    config5,
    random_tiny,
    CONFIG_NAMES,
)
