"""Small k_dst_lvl4 run for compute-sanitizer: python tools/lvl4_debug.py [L]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np
import torch
import paper_2107_06381_b200 as B
from oracle import bhcp_oracle as O
from paper_2107_06381_b200.space import plan_for
from test_gpu_levels import blocked, run_levels, rel

L = int(sys.argv[1]) if len(sys.argv) > 1 else 1
m = 1023
plan = plan_for(B.build_grid(2, 1.0, 1024))
rng = np.random.default_rng(5)
F = rng.standard_normal((L, m * m))
ref = O.fused_pass_b(F, 2, m)
W = blocked(F, 2, m)
y = run_levels(plan.handle, W, L, 2, m, "fused")
print("L", L, "finite", np.isfinite(y).all(), "rel", rel(y, ref))
