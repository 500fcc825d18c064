"""Regularisation-parameter sweep: BASELINE config c5's error-vs-alpha curve.

c5 is 128 independent solves of one g_delta: 64 log-spaced alpha in
[1e-6, 1e-1] for each of pint-qbvm and pint-mqbvm. Every solve reports the
reconstruction error e_h = l2_error(y[0], z0) of the reference driver
(bench.py:154-162; the curve the driver builds from one row per alpha,
bench.py:265-271). Multi-GPU is replicas: rank r takes the
(kind, alpha) pairs i = r, r + P, ... and the 128 scalars are gathered on
every rank. No collective on the data path.

Per solve on the device: the plan for that (kind, alpha) -- its omega sets
Gamma and the shifts, so the host tables (diagonalize, pint.py:87) are built
per pair, while the next pair's tables are built as the current solve runs --
then the fused solve, then y[0] (one level) back to the host.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import Callable, List, Sequence, Tuple

import numpy as np


@dataclass
class SweepPoint:
    kind: str
    alpha: float
    e_h: float
    ms: float          # device time of the solve (CUDA events)
    rank: int


@dataclass
class SweepResult:
    points: List[SweepPoint] = field(default_factory=list)
    wall_s: float = 0.0    # max over ranks

    def curve(self, kind: str) -> Tuple[np.ndarray, np.ndarray]:
        pts = sorted((p for p in self.points if p.kind == kind), key=lambda p: p.alpha)
        return np.array([p.alpha for p in pts]), np.array([p.e_h for p in pts])

    def best(self, kind: str) -> SweepPoint:
        return min((p for p in self.points if p.kind == kind), key=lambda p: p.e_h)


def assign(n_pairs: int, rank: int, world: int) -> List[int]:
    """Pairs of this rank: i = rank, rank + world, ... (round robin; every
    solve costs the same, so the ranks are balanced to one solve)."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    return list(range(rank, n_pairs, world))


def gather(local: List[SweepPoint], world: int, comm=None) -> List[SweepPoint]:
    """All ranks' points, in pair order (torch.distributed all_gather_object)."""
    if world == 1:
        return list(local)
    import torch.distributed as dist

    parts: list = [None] * world
    dist.all_gather_object(parts, [(p.kind, p.alpha, p.e_h, p.ms, p.rank) for p in local], group=comm)
    out = [SweepPoint(*t) for part in parts for t in part]
    return out


def run_pairs(pairs: Sequence[Tuple[str, float]], solve_one: Callable[[str, float], Tuple[float, float]],
              rank: int = 0, world: int = 1, comm=None) -> SweepResult:
    """Host orchestration: solve this rank's pairs with `solve_one(kind, alpha)
    -> (e_h, ms)`, gather every rank's points, wall time = max over ranks."""
    t0 = time.perf_counter()
    local = []
    for i in assign(len(pairs), rank, world):
        kind, alpha = pairs[i]
        e_h, ms = solve_one(kind, alpha)
        local.append(SweepPoint(kind, float(alpha), float(e_h), float(ms), rank))
    wall = time.perf_counter() - t0
    pts = gather(local, world, comm)
    if world > 1:
        import torch
        import torch.distributed as dist

        dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(comm) == "nccl" else "cpu"
        w = torch.tensor([wall], dtype=torch.float64, device=dev)
        dist.all_reduce(w, op=dist.ReduceOp.MAX, group=comm)
        wall = float(w.item())
    order = {(k, float(a)): j for j, (k, a) in enumerate(pairs)}
    pts.sort(key=lambda p: order[(p.kind, p.alpha)])
    return SweepResult(pts, wall)


def alpha_sweep(grid, timegrid, g_delta, z0, kinds: Sequence[str], alphas: Sequence[float],
                rank: int = 0, world: int = 1, comm=None) -> SweepResult:
    """The device sweep: one fused solve per (kind, alpha) on this rank's GPU."""
    import torch

    from . import _lib, methods, pint, plans
    from .workloads import l2_error

    _lib.lib()   # fails loudly without the CUDA library / a GPU
    g_dev = plans.to_device(np.asarray(g_delta, dtype=np.float64), torch.float64)
    y = torch.empty((timegrid.n_levels, grid.n_interior), dtype=torch.float64, device=g_dev.device)
    pairs = [(k, float(a)) for k in kinds for a in alphas]

    def build(kind, alpha):
        system = methods.assemble(methods.MethodKind(kind), alpha, grid, timegrid, g_delta)
        plan = pint.PintPlan(grid, timegrid.n_levels, timegrid.tau, system.omega)
        return plan, system.method.condition_divisor(timegrid.tau)

    mine = [pairs[i] for i in assign(len(pairs), rank, world)]
    built = {}
    if mine:
        built[mine[0]] = build(*mine[0])
    ws_shared = [None]

    def solve_one(kind, alpha):
        plan, div = built.pop((kind, alpha))
        if ws_shared[0] is None:
            ws_shared[0] = plan.workspace()
        plan.use_workspace(ws_shared[0])   # every (kind, alpha) plan has the same workspace size
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.solve_device(g_dev, div, out=y)
        e1.record()
        # the next pair's host tables are built while this solve runs
        j = mine.index((kind, alpha))
        if j + 1 < len(mine):
            built[mine[j + 1]] = build(*mine[j + 1])
        y0 = y[0].cpu().numpy()          # synchronises
        plan.check_status()
        return l2_error(y0, z0, grid.h, grid.dim), e0.elapsed_time(e1)

    return run_pairs(pairs, solve_one, rank, world, comm)
