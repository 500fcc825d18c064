"""Parallel-in-time direct solve of the pint-qbvm / pint-mqbvm systems on the
B200 (mirrors pkg/src/bhcp/pint.py).

solve_pint (pint.py:69-110) computes the trajectory of the all-at-once system
B y = rhs with B = Gamma^{-1} F* D F Gamma (block omega-circulant). The
reference applies, along time and space,

    (a) S1 = F Gamma rhs               time FFT of the Gamma-scaled rhs
    (b) S2[:, j] = (s_j - lap)^{-1} S1[:, j] = Phi diag(1/(s_j + mu)) Phi S1[:, j]
    (c) y = Re Gamma^{-1} F* S2        time FFT back, residue check

with Phi the orthonormal (involutory, real) DST-I. The device path performs
the same linear maps with the inverse spatial transform moved after the time
transform -- Phi acts on space and F, Gamma, Re act on time, so they commute:

    ghat     = Phi g / (divisor * n)                         [bhcp_pint_ghat]
    W[t, k]  = ghat_k Re( Gamma^{-1}_t sum_j e^{-2 pi i jt/n} / (s_j + mu_k) )
                                                             [bhcp_pint_modes]
    y[t, :]  = Phi W[t, :]                                   [bhcp_pint_levels]

Step (a) needs no time FFT on device because rhs is nonzero only in block 0
and gamma_0 = 1 (methods.py:158-162, circulant.py:148), so every column of S1
equals rhs_0 / sqrt(n) and one forward DST serves all levels. The imaginary
residue of (c) is measured on the mode coefficients, where it has the same
Frobenius norm because Phi is orthonormal. The literal
3-step dataflow is ``solve_pint_unfused`` (same kernels family) and is checked
against the fused path in tests.
"""

from __future__ import annotations

import ctypes
from typing import Optional

import numpy as np
import torch

from . import _lib
from . import plans
from .circulant import ImaginaryResidueError, diagonalize
from .methods import SolveResult, condition_divisor
from .space import SingularShiftError, SpatialGrid, mu1_of, plan_for, singular_message, solve_levels

RESIDUE_TOL = 1e-8  # circulant.py:170


def step_b_parallel(grid: SpatialGrid, block, shifts, backend: str = "spectral", workers: Optional[int] = None):
    """Solve (shifts[j] I - lap) x_j = block[:, j] for every column j (pint.py:26-66).

    All columns are solved by one batched device launch sequence; results are
    bit-identical for any ``workers`` value (accepted for compatibility).
    """
    is_torch = isinstance(block, torch.Tensor)
    shape = tuple(block.shape) if is_torch else np.asarray(block).shape
    shifts = np.atleast_1d(np.asarray(shifts))
    if len(shape) != 2 or shape[1] != shifts.shape[0]:
        raise ValueError(f"need one shift per column, got block {shape} and {shifts.shape[0]} shifts")
    if backend not in ("spectral", "banded"):
        raise ValueError(f"unknown backend {backend!r}")
    n_space, n_cols = shape
    if n_space != grid.n_interior:
        raise ValueError(f"rhs must have shape ({grid.n_interior},), got ({n_space},)")
    src = plans.to_device(block, torch.complex128)
    levels = plans.transpose(src, n_space, n_cols)  # (n_cols, n_space) level-major
    out, bad = solve_levels(grid, levels, shifts.astype(np.complex128))
    if bad >= 0:
        raise SingularShiftError(f"column {bad}: {singular_message(complex(shifts[bad]))}")
    res = plans.transpose(out, n_cols, n_space)
    return res if is_torch else res.cpu().numpy()


class PintPlan:
    """Device plans + workspace for repeated solves of one (grid, time grid, omega)."""

    def __init__(self, grid: SpatialGrid, n_levels: int, tau: float, omega: float):
        self.grid = grid
        self.n = n_levels
        self.tau = tau
        self.diag = diagonalize(n_levels, omega)            # pint.py:87, untimed
        self.shifts = self.diag.eigenvalues / tau            # pint.py:95
        self.sp = plan_for(grid)
        self.tp = plans.time_plan(self.diag.gamma, self.shifts)
        lib = _lib.lib()
        self.ws_bytes = int(lib.bhcp_pint_workspace_bytes(self.sp.handle, self.tp.handle))
        self._ws: Optional[torch.Tensor] = None

    def use_workspace(self, ws: torch.Tensor) -> None:
        """Share a workspace between plans of the same grid and level count (their
        sizes agree; e.g. the plans of an alpha sweep). The caller serialises the
        solves that use it."""
        if ws.numel() < self.ws_bytes or ws.dtype != torch.uint8:
            raise ValueError(f"workspace of {ws.numel()} bytes, this plan needs {self.ws_bytes}")
        self._ws = ws

    def workspace(self) -> torch.Tensor:
        if self._ws is None:
            self._ws = torch.empty(self.ws_bytes, dtype=torch.uint8,
                                   device=torch.device("cuda", torch.cuda.current_device()))
        return self._ws

    def solve_device(self, g: torch.Tensor, divisor: float, out: Optional[torch.Tensor] = None,
                     events: Optional[list] = None) -> torch.Tensor:
        """Enqueue the fused solve on the current stream; returns y (n, n_space).

        ``events`` (4 torch CUDA events) are recorded at the phase boundaries.
        Status is read separately with ``check_status``.
        """
        lib = _lib.lib()
        nx = self.grid.n_interior
        y = out if out is not None else torch.empty((self.n, nx), dtype=torch.float64, device=g.device)
        ws = self.workspace()
        stream = plans.stream_handle()
        wsp = ws.data_ptr()
        status = ctypes.c_void_p(lib.bhcp_pint_status_ptr(self.sp.handle, self.tp.handle, ctypes.c_void_p(wsp)))
        if not events:
            # one call: status reset, ghat, pass A (the 1/(divisor n) scale folded into
            # its coefficients) and the level passes
            _lib.check(lib.bhcp_pint_solve(self.sp.handle, self.tp.handle, plans.ptr(g), divisor, plans.ptr(y),
                                           ctypes.c_void_p(wsp), self.ws_bytes, stream), "bhcp_pint_solve")
            return y
        ghat = ctypes.c_void_p(wsp + 256)
        W = ctypes.c_void_p(wsp + 256 + ((8 * nx + 255) // 256) * 256)
        if events:
            events[0].record()
        _lib.check(lib.bhcp_status_reset(status, stream), "bhcp_status_reset")
        _lib.check(lib.bhcp_pint_ghat(self.sp.handle, plans.ptr(g), 1.0 / (divisor * self.n), ghat, stream),
                   "bhcp_pint_ghat")
        if events:
            events[1].record()
        _lib.check(lib.bhcp_pint_modes(self.sp.handle, self.tp.handle, ghat, 0, nx, W, 0, None, status, stream),
                   "bhcp_pint_modes")
        if events:
            events[2].record()
        # the level phase exactly as bhcp_pint_solve runs it: the level-group kernel
        # where the plan has one, its scratch in the workspace right after W
        nw = nx * 8 * ((self.n + 7) // 8)
        sync = ctypes.c_void_p(W.value + ((8 * nw + 255) // 256) * 256)
        _lib.check(lib.bhcp_pint_levels_fused(self.sp.handle, W, plans.ptr(y), self.n, sync, stream),
                   "bhcp_pint_levels_fused")
        if events:
            events[3].record()
        return y

    def capture(self, g: torch.Tensor, divisor: float, out: torch.Tensor) -> "torch.cuda.CUDAGraph":
        """Capture one fused solve (g -> out, fixed buffers) into a CUDA graph;
        ``graph.replay()`` then re-runs status reset, ghat, pass A and the level
        passes with a single launch from the host. Plans are immutable (every
        device table, symmetric tile lists included, is built at plan
        creation), so a fresh plan captures without an eager solve first."""
        self.workspace()
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            with torch.cuda.graph(graph, stream=side):
                self.solve_device(g, divisor, out=out)
        torch.cuda.current_stream().wait_stream(side)
        return graph

    def status_ptr(self) -> ctypes.c_void_p:
        ws = self.workspace()
        return ctypes.c_void_p(ws.data_ptr())

    def read_status(self, tol: float = RESIDUE_TOL, status: Optional[ctypes.c_void_p] = None) -> _lib.Status:
        """The status block of the last solve (synchronises): code, first singular
        column, ||Im Y|| (residue) and ||Y|| (norm) of circulant.py:182-185.
        ``status``: another status block written for this plan (a batched solve)."""
        st = _lib.Status()
        ptr = status if status is not None else self.status_ptr()
        _lib.check(_lib.lib().bhcp_read_status(ptr, tol, ctypes.byref(st), plans.stream_handle()),
                   "bhcp_read_status")
        return st

    def check_status(self, tol: float = RESIDUE_TOL, status: Optional[ctypes.c_void_p] = None) -> _lib.Status:
        st = self.read_status(tol, status)
        if st.code == _lib.BHCP_ERR_SINGULAR_SHIFT:
            j = int(st.bad_column)
            raise SingularShiftError(f"column {j}: {singular_message(complex(self.shifts[j]))}")
        if st.code == _lib.BHCP_ERR_IMAGINARY_RESIDUE:
            raise ImaginaryResidueError(
                f"imaginary residue {st.residue:.3e} exceeds {tol:.1e} of the result norm {st.norm:.3e}"
            )
        return st

    def solve_unfused_device(self, g: torch.Tensor, divisor: float, out: Optional[torch.Tensor] = None):
        """Literal 3-step dataflow (pint.py:89-99) on the device; returns (y, status tensor)."""
        lib = _lib.lib()
        nx = self.grid.n_interior
        y = out if out is not None else torch.empty((self.n, nx), dtype=torch.float64, device=g.device)
        nb = int(lib.bhcp_pint_unfused_workspace_bytes(self.sp.handle, self.tp.handle))
        ws = torch.empty(nb, dtype=torch.uint8, device=g.device)
        _lib.check(lib.bhcp_pint_solve_unfused(self.sp.handle, self.tp.handle, plans.ptr(g), divisor, plans.ptr(y),
                                               plans.ptr(ws), nb, plans.stream_handle()),
                   "bhcp_pint_solve_unfused")
        return y, ws


class PintBatch:
    """Independent fused solves of one g on one grid and time length, each with
    its own (kind, alpha) plan (BASELINE config 5: the alpha sweep), enqueued as
    one batched call (``bhcp_pint_solve_batch``): one DST of g, pass A of up to
    32 solves per launch, one level phase for all. No host synchronisation; the
    status blocks are read with ``check(i)``. Each trajectory is bitwise the one
    ``PintPlan.solve_device`` gives for that plan."""

    def __init__(self, plans_: "list[PintPlan]", ws: Optional[torch.Tensor] = None):
        if not plans_:
            raise ValueError("empty batch")
        n = plans_[0].n
        if any(p.n != n or p.grid != plans_[0].grid for p in plans_):
            raise ValueError("a batch needs one grid and one number of levels")
        self.plans = list(plans_)
        self.nb = len(self.plans)
        lib = _lib.lib()
        self.sp = self.plans[0].sp
        self.ws_bytes = int(lib.bhcp_pint_batch_workspace_bytes(self.sp.handle, self.plans[0].tp.handle, self.nb))
        dev = torch.device("cuda", torch.cuda.current_device())
        if ws is not None and (ws.dtype != torch.uint8 or ws.numel() < self.ws_bytes):
            raise ValueError(f"workspace of {ws.numel()} bytes, this batch needs {self.ws_bytes}")
        # a shared workspace is reused in stream order (the caller serialises the batches)
        self.ws = ws if ws is not None else torch.empty(self.ws_bytes, dtype=torch.uint8, device=dev)
        self.sbytes = int(lib.bhcp_status_bytes())
        self.status = torch.empty(self.nb * self.sbytes, dtype=torch.uint8, device=dev)
        self._tps = (ctypes.c_void_p * self.nb)(*[p.tp.handle.value for p in self.plans])

    def solve_device(self, g: torch.Tensor, divisors, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Enqueue every solve; returns y (nb, n, n_space)."""
        lib = _lib.lib()
        nx = self.plans[0].grid.n_interior
        y = out if out is not None else torch.empty((self.nb, self.plans[0].n, nx), dtype=torch.float64,
                                                    device=g.device)
        div = (ctypes.c_double * self.nb)(*[float(d) for d in divisors])
        _lib.check(lib.bhcp_pint_solve_batch(self.sp.handle, self._tps, self.nb, plans.ptr(g), div, plans.ptr(y),
                                             plans.ptr(self.status), plans.ptr(self.ws), self.ws_bytes,
                                             plans.stream_handle()), "bhcp_pint_solve_batch")
        return y

    def check(self, i: int, tol: float = RESIDUE_TOL) -> _lib.Status:
        """Status of solve i (synchronises); raises like ``PintPlan.check_status``."""
        return self.plans[i].check_status(tol, ctypes.c_void_p(self.status.data_ptr() + i * self.sbytes))


_plan_cache: dict = {}


def pint_plan(grid: SpatialGrid, timegrid, omega: float) -> PintPlan:
    key = (torch.cuda.current_device(), grid, timegrid.n_levels, timegrid.tau, float(omega))
    plan = _plan_cache.get(key)
    if plan is None:
        if len(_plan_cache) > 16:
            _plan_cache.clear()
        plan = PintPlan(grid, timegrid.n_levels, timegrid.tau, omega)
        _plan_cache[key] = plan
    return plan


def _check_kind(system) -> None:
    kind = system.method.kind
    if not kind.is_circulant:
        raise ValueError(f"{kind.value} has no circulant time coupling; use the sparse baseline")


def solve_pint(system, backend: str = "spectral", workers: Optional[int] = None) -> SolveResult:
    """Solve a circulant-kind all-at-once system by FFT diagonalisation (pint.py:69-110).

    Returns a SolveResult whose ``trajectory`` is the (n_levels, n_space)
    float64 C-contiguous host array (copied from HBM on first access) and
    whose ``trajectory_device`` is the device tensor. ``timings`` holds the
    CUDA-event durations of the three phases under the reference's keys
    (step_a = forward spatial transform of the data, step_b = shifted divides +
    time transform, step_c = inverse spatial transform + residue check) and
    their sum as ``total``. ``backend`` and ``workers`` are accepted for
    signature compatibility; the device path is deterministic.
    """
    _check_kind(system)
    if backend not in ("spectral", "banded"):
        raise ValueError(f"unknown backend {backend!r}")
    _lib.lib()  # raises NativeLibraryError when the CUDA library cannot run here
    tau = system.timegrid.tau
    plan = pint_plan(system.grid, system.timegrid, system.omega)
    divisor = condition_divisor(system.method.kind, system.method.alpha, tau)
    g = plans.to_device(system.data, torch.float64)
    events = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    y = plan.solve_device(g, divisor, events=events)
    st = plan.check_status()  # synchronises; raises under circulant.py:182-189
    t_a = events[0].elapsed_time(events[1]) / 1e3
    t_b = events[1].elapsed_time(events[2]) / 1e3
    t_c = events[2].elapsed_time(events[3]) / 1e3
    timings = {"step_a": t_a, "step_b": t_b, "step_c": t_c, "total": t_a + t_b + t_c}
    res = SolveResult(system=system, trajectory=None, solver="pint", timings=timings, trajectory_device=y)
    res.residue_ratio = float(st.residue / st.norm) if st.norm > 0 else 0.0   # ||Im Y|| / ||Y||
    return res


def solve_pint_unfused(system) -> SolveResult:
    """The reference's literal 3-step dataflow on the device (rhs block, time
    FFT, per-level shifted solves, time FFT back), for validation of the fused
    path and for the bench's dataflow comparison."""
    _check_kind(system)
    tau = system.timegrid.tau
    plan = pint_plan(system.grid, system.timegrid, system.omega)
    divisor = condition_divisor(system.method.kind, system.method.alpha, tau)
    g = plans.to_device(system.data, torch.float64)
    y, ws = plan.solve_unfused_device(g, divisor)
    st = _lib.Status()
    _lib.check(_lib.lib().bhcp_read_status(plans.ptr(ws), RESIDUE_TOL, ctypes.byref(st), plans.stream_handle()),
               "bhcp_read_status")
    if st.code == _lib.BHCP_ERR_SINGULAR_SHIFT:
        j = int(st.bad_column)
        raise SingularShiftError(f"column {j}: {singular_message(complex(plan.shifts[j]))}")
    if st.code == _lib.BHCP_ERR_IMAGINARY_RESIDUE:
        raise ImaginaryResidueError(
            f"imaginary residue {st.residue:.3e} exceeds {RESIDUE_TOL:.1e} of the result norm {st.norm:.3e}"
        )
    return SolveResult(system=system, trajectory=None, solver="pint-unfused", timings={}, trajectory_device=y)


def device_residual_norm(system, y_dev: torch.Tensor) -> float:
    """||rhs - A y|| / ||rhs|| on the device for a pint-kind system
    (methods.py:239-247)."""
    _check_kind(system)
    lib = _lib.lib()
    sp = plan_for(system.grid)
    tau = system.timegrid.tau
    divisor = condition_divisor(system.method.kind, system.method.alpha, tau)
    g = plans.to_device(system.data, torch.float64)
    ws = torch.empty(int(lib.bhcp_residual_workspace_bytes()), dtype=torch.uint8, device=y_dev.device)
    out = (ctypes.c_double * 2)()
    _lib.check(lib.bhcp_residual_norm(sp.handle, plans.ptr(y_dev), system.n_levels, tau, divisor, system.grid.h,
                                      plans.ptr(g), plans.ptr(ws), out, plans.stream_handle()), "bhcp_residual_norm")
    return float(out[0] / out[1]) if out[1] > 0 else float(out[0])
