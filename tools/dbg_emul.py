import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, torch
import paper_2107_06381_b200 as B
from paper_2107_06381_b200 import workloads
from test_distributed import emulate
for dim, cells, steps, world in [(2, 20, 9, 1), (2, 20, 9, 2), (2, 20, 9, 3), (2, 16, 12, 2)]:
    w = workloads.make_small(dim, cells, steps, seed=3)
    grid = B.build_grid(dim, w.length, cells); tg = B.TimeGrid(w.horizon, steps)
    system = B.assemble(B.MethodKind.PINT_MQBVM, 1e-2, grid, tg, w.g_delta)
    single = B.solve_pint(system).trajectory
    multi = emulate(system, world)
    d = np.abs(single - multi)
    idx = np.unravel_index(d.argmax(), d.shape)
    print(dim, cells, steps, world, d.max(), np.abs(single).max(), idx, (d > 0).sum(), d.shape)
    if d.max() > 0:
        bad_levels = sorted(set(np.nonzero(d)[0].tolist()))
        print('  bad levels', bad_levels[:20])
