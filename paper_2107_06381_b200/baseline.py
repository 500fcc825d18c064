"""Closed-form solver and forward model on the device (mirrors the parts of
pkg/src/bhcp/baseline.py that the PinT path's callers use).

``solve_spectral_oracle`` (baseline.py:67-112) is the reference's exact
per-mode solve. It is a separate solver -- the reference itself says it is
not to be benchmarked as the PinT solver -- and ``solve_pint`` never calls it.
Here it serves full-size verification on the GPU and as the
device counterpart of the reference's ``--solver oracle`` path.
``march_forward`` (baseline.py:115-129) generates final data g from an
initial state with the per-mode identity g = DST(rho^N DST(z0)) (f2).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib, plans
from .methods import AllAtOnceSystem, MethodSpec, SolveResult
from .space import SpatialGrid, plan_for

_KIND_CODE = {"qbvm": 0, "mqbvm": 1, "pint-qbvm": 2, "pint-mqbvm": 3}


def solve_spectral_oracle(kind, alpha: float, grid: SpatialGrid, timegrid, data) -> SolveResult:
    """Closed-form per-mode solve of any of the four methods (baseline.py:67-112)."""
    data = np.asarray(data, dtype=float) if not isinstance(data, torch.Tensor) else data
    if tuple(data.shape) != (grid.n_interior,):
        raise ValueError(f"final data must have shape ({grid.n_interior},), got {tuple(data.shape)}")
    lib = _lib.lib()
    sp = plan_for(grid)
    n = timegrid.n_levels
    g = plans.to_device(data, torch.float64)
    y = torch.empty((n, grid.n_interior), dtype=torch.float64, device=g.device)
    nb = int(lib.bhcp_spectral_workspace_bytes(sp.handle, n))
    ws = torch.empty(nb, dtype=torch.uint8, device=g.device)
    code = _KIND_CODE[kind.value if hasattr(kind, "value") else str(kind)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    _lib.check(lib.bhcp_spectral_solve(sp.handle, code, float(alpha), timegrid.tau, timegrid.num_steps, plans.ptr(g),
                                       plans.ptr(y), plans.ptr(ws), nb, plans.stream_handle()), "bhcp_spectral_solve")
    stop.record()
    stop.synchronize()
    system = AllAtOnceSystem(MethodSpec(kind, alpha), grid, timegrid, np.asarray(data.cpu() if isinstance(data, torch.Tensor) else data))
    return SolveResult(system=system, trajectory=None, solver="spectral-oracle",
                       timings={"total": start.elapsed_time(stop) / 1e3}, trajectory_device=y)


def march_forward(initial, timegrid, grid: SpatialGrid):
    """Backward Euler recursion of the initial state to t = T (baseline.py:115-129),
    computed per mode as DST(rho^N DST(z0)) on the device."""
    is_torch = isinstance(initial, torch.Tensor)
    z0 = plans.to_device(initial, torch.float64)
    if tuple(z0.shape) != (grid.n_interior,):
        raise ValueError(f"initial state must have shape ({grid.n_interior},), got {tuple(z0.shape)}")
    sp = plan_for(grid)
    out = torch.empty_like(z0)
    _lib.check(_lib.lib().bhcp_march_forward(sp.handle, timegrid.tau, timegrid.num_steps, plans.ptr(z0), plans.ptr(out),
                                             plans.stream_handle()), "bhcp_march_forward")
    return out if is_torch else out.cpu().numpy()
