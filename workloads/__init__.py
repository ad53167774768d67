"""Seeded synthetic PPipe planning workloads (input recipe only).

This package is shared by the CPU oracle tests and the CUDA path. It holds
only input generation (profile tables, feature-map sizes, bandwidth matrix,
SLOs); none of the method's arithmetic (stage latency, transfer time, E2E
latency, feasibility, throughput, frontier) lives here. See DESIGN.md
"Input recipe" and SURVEY.md §8(d).
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
