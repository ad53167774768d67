"""CPU oracle for the PPipe plan-enumeration hot path.

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package. The product
package (paper_2507_18748_b200) never imports it and shares no code with it.
"""
from .oracle import (  # noqa: F401
    POINT_DTYPE,
    POINT_PB_DTYPE,
    OracleResult,
    build_oracle,
    run_oracle,
    run_oracle_pb,
    oracle_lib_path,
    prepartition_oracle,
)
