"""Small workloads through the product path, for compute-sanitizer runs."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2507_18748_b200 as pp
from workloads import make_config, random_tiny

for cfg in (1, 2, 3):
    g = pp.run(make_config(cfg), device=0)
    print("config", cfg, g.n_points, flush=True)
w = make_config(5, n_models=2)
g = pp.run(w, device=0)
print("config 5 x2", g.n_points, flush=True)
for seed in range(20):
    g = pp.run(random_tiny(seed), device=0)
print("tiny ok", flush=True)
# shard mode (world > 1 without NCCL): rank 1 of 3
g = pp.run(make_config(3), rank=1, world=3, device=0)
print("shard ok", g.n_points, flush=True)
