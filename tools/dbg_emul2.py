import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, torch
import paper_2107_06381_b200 as B
from paper_2107_06381_b200 import workloads
from test_distributed import emulate
w = workloads.make("c2")
grid = B.build_grid(2, w.length, w.num_cells); tg = B.TimeGrid(w.horizon, w.num_steps)
system = B.assemble(B.MethodKind.PINT_MQBVM, 1e-2, grid, tg, w.g_delta)
single = B.solve_pint(system).trajectory
for world in (1, 2, 8):
    multi = emulate(system, world)
    d = np.abs(single - multi)
    print(world, d.max(), np.linalg.norm(single - multi) / np.linalg.norm(single), (d > 0).sum())
    if d.max() > 0:
        lv = sorted(set(np.nonzero(d)[0].tolist()))
        print('  levels', lv[:10], len(lv))
        sp = np.nonzero(d[lv[0]])[0]
        print('  positions in level', lv[0], sp[:10], len(sp))
