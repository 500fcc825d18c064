"""Run a few fused c2 solves (for ncu captures): python tools/profile_step.py [config] [reps]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2107_06381_b200 as B
from paper_2107_06381_b200 import workloads

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
w = workloads.make(name)
grid = B.build_grid(w.dim, w.length, w.num_cells)
tg = B.TimeGrid(w.horizon, w.num_steps)
system = B.assemble(B.MethodKind(w.kinds[0]), w.alphas[0], grid, tg, w.g_delta)
plan = B.PintPlan(grid, tg.n_levels, tg.tau, system.omega)
g = torch.from_numpy(w.g_delta).cuda()
div = system.method.condition_divisor(tg.tau)
y = plan.solve_device(g, div)
for _ in range(reps):
    plan.solve_device(g, div, out=y)
torch.cuda.synchronize()
plan.check_status()
print("ok", name, float(y[0].abs().max()))
