import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, torch
import paper_2107_06381_b200 as B
from paper_2107_06381_b200.space import plan_for
from test_gpu_levels import blocked, run_levels
m = 1023
plan = plan_for(B.build_grid(2, 1.0, 1024))
rng = np.random.default_rng(5)
F = rng.standard_normal((20, m * m))
y20 = run_levels(plan.handle, blocked(F, 2, m), 20, 2, m, "fused")
y8 = run_levels(plan.handle, blocked(F[:8], 2, m), 8, 2, m, "fused")
y9 = run_levels(plan.handle, blocked(F[:9], 2, m), 9, 2, m, "fused")
for name, a, b in (("8 vs 20", y8, y20[:8]), ("9 vs 20", y9, y20[:9])):
    d = np.abs(a - b)
    print(name, "rel", np.linalg.norm(a - b) / np.linalg.norm(b), "levels differing", [int(t) for t in np.nonzero(d.max(axis=1))[0]])
    if d.max() > 0:
        t = int(np.argmax(d.max(axis=1))); dd = d[t].reshape(m, m); r, c = np.nonzero(dd)
        print("  level", t, "rows", np.unique(r)[:8], "n", len(r), "cols", np.unique(c)[:8])
