"""Regularisation-parameter sweep: BASELINE config c5's error-vs-alpha curve.

c5 is 128 independent solves of one g_delta: 64 log-spaced alpha in
[1e-6, 1e-1] for each of pint-qbvm and pint-mqbvm. Every solve reports the
reconstruction error e_h = l2_error(y[0], z0) of the reference driver
(bench.py:154-162; the curve the driver builds from one row per alpha,
bench.py:265-271). Multi-GPU is replicas: rank r takes the
(kind, alpha) pairs i = r, r + P, ... and the 128 scalars are gathered on
every rank. No collective on the data path.

On the device the pairs run batched (``pint.PintBatch``): each (kind, alpha)
keeps its own plan (its omega sets Gamma and the shifts, the host tables of
diagonalize, pint.py:87), a chunk of solves is one ``bhcp_pint_solve_batch``
call (one DST of g, pass A of the whole chunk per launch, one level phase),
e_h of each solve is reduced on the device, and the host synchronises once.
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
                rank: int = 0, world: int = 1, comm=None, chunk: int = 16) -> SweepResult:
    """The device sweep: this rank's (kind, alpha) pairs as batched fused solves
    (``pint.PintBatch``, ``chunk`` solves per call), e_h of every solve reduced on
    the device, one host synchronisation at the end."""
    import torch

    from . import _lib, methods, pint, plans

    _lib.lib()   # fails loudly without the CUDA library / a GPU
    g_dev = plans.to_device(np.asarray(g_delta, dtype=np.float64), torch.float64)
    z0_dev = plans.to_device(np.asarray(z0, dtype=np.float64), torch.float64)
    pairs = [(k, float(a)) for k in kinds for a in alphas]
    mine = [pairs[i] for i in assign(len(pairs), rank, world)]
    t0 = time.perf_counter()
    local: List[SweepPoint] = []
    if mine:
        nb = min(chunk, len(mine))
        y = torch.empty((nb, timegrid.n_levels, grid.n_interior), dtype=torch.float64, device=g_dev.device)
        e_h = torch.empty(len(mine), dtype=torch.float64, device=g_dev.device)
        scale = float(np.sqrt(grid.h ** grid.dim))   # l2_error (bench.py:154-162)
        batches, events = [], []
        ws = None
        for c0 in range(0, len(mine), nb):
            c1 = min(c0 + nb, len(mine))
            # this chunk's plans (host tables of diagonalize, pint.py:87) are built
            # while the previous chunk runs on the device
            systems = [methods.assemble(methods.MethodKind(k), a, grid, timegrid, g_delta) for k, a in mine[c0:c1]]
            b = pint.PintBatch([pint.PintPlan(grid, timegrid.n_levels, timegrid.tau, sy.omega) for sy in systems], ws)
            ws = b.ws   # one workspace for every chunk (stream order)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            yb = b.solve_device(g_dev, [sy.method.condition_divisor(timegrid.tau) for sy in systems], out=y[: c1 - c0])
            e1.record()
            # e_h = sqrt(h^dim) ||y(0) - z0|| of every solve, before y is reused
            e_h[c0:c1] = torch.linalg.vector_norm(yb[:, 0, :] - z0_dev, dim=1) * scale
            batches.append((c0, b))
            events.append((e0, e1, c1 - c0))
        e_host = e_h.cpu().numpy()   # the one synchronisation
        for c0, b in batches:
            for i in range(b.nb):
                b.check(i)
        for (c0, b), (e0, e1, cnt) in zip(batches, events):
            ms = e0.elapsed_time(e1) / cnt
            for i in range(cnt):
                k, a = mine[c0 + i]
                local.append(SweepPoint(k, a, float(e_host[c0 + i]), ms, rank))
    wall = time.perf_counter() - t0
    pts = gather(local, world, comm)
    if world > 1:
        import torch.distributed as dist

        dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(comm) == "nccl" else "cpu"
        w = torch.tensor([wall], dtype=torch.float64, device=dev)
        dist.all_reduce(w, op=dist.ReduceOp.MAX, group=comm)
        wall = float(w.item())
    order = {(k, float(a)): j for j, (k, a) in enumerate(pairs)}
    pts.sort(key=lambda p: order[(p.kind, p.alpha)])
    return SweepResult(pts, wall)
