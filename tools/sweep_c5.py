"""BASELINE config 5 on one GPU: the full 128-solve error-vs-alpha sweep,
batched (sweep.alpha_sweep), timed twice (the first pass builds and caches the
128 time plans). Prints one JSON object: device ms (sum of the batch events),
wall s, and the largest relative e_h deviation from the closed-form oracle.
usage: python tools/sweep_c5.py [chunk]"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_2107_06381_b200 as B
from oracle import bhcp_oracle as O
from paper_2107_06381_b200 import sweep, workloads

chunk = int(sys.argv[1]) if len(sys.argv) > 1 else 16
w = workloads.make("c5")
grid = B.build_grid(w.dim, w.length, w.num_cells)
tg = B.TimeGrid(w.horizon, w.num_steps)
runs = []
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = sweep.alpha_sweep(grid, tg, w.g_delta, w.z0, w.kinds, w.alphas, chunk=chunk)
    wall = time.perf_counter() - t0
    dev_ms = sum(p.ms for p in res.points)
    runs.append({"wall_s": wall, "device_ms": dev_ms})
dev = 0.0
worst = None
for p in res.points:
    ref = O.spectral_oracle(p.kind, p.alpha, w.dim, w.length, w.num_cells, w.horizon, w.num_steps, w.g_delta,
                            levels=np.array([0]))
    e_ref = workloads.l2_error(ref[0], w.z0, grid.h, w.dim)
    d = abs(p.e_h - e_ref) / e_ref
    if d > dev:
        dev, worst = d, (p.kind, p.alpha)
best = {k: (res.best(k).alpha, res.best(k).e_h) for k in w.kinds}
print(json.dumps({"config": "c5", "solves": len(res.points), "chunk": chunk, "runs": runs,
                  "max_rel_dev_e_h": dev, "worst": worst, "best": best,
                  "curve": {k: [list(map(float, v)) for v in res.curve(k)] for k in w.kinds}}))
