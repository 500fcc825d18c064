"""Method kinds, the all-at-once system and the solve result (mirrors
pkg/src/bhcp/methods.py for the pieces the PinT path uses).

The sparse explicit operator (methods.py:173-190) serves only the reference's
sparse-LU comparator, which is out of scope here.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass
from typing import Optional

import numpy as np

from .circulant import TimeGrid
from .space import LaplacianOperator, SpatialGrid


class MethodKind(enum.Enum):
    """The four regularisation methods; values double as CLI tokens (methods.py:34-45)."""

    QBVM = "qbvm"
    MQBVM = "mqbvm"
    PINT_QBVM = "pint-qbvm"
    PINT_MQBVM = "pint-mqbvm"

    @property
    def is_circulant(self) -> bool:
        return self in (MethodKind.PINT_QBVM, MethodKind.PINT_MQBVM)


def _kind_value(kind) -> str:
    return kind.value if hasattr(kind, "value") else str(kind)


def alpha_rule(kind, delta: float, tau: float, fallback: float = 1e-12, e0: Optional[float] = None) -> float:
    """methods.py:48-71."""
    if delta < 0:
        raise ValueError(f"noise magnitude must be nonnegative, got {delta}")
    if tau <= 0:
        raise ValueError(f"time step must be positive, got {tau}")
    if delta == 0:
        return fallback
    if e0 is not None:
        delta = delta / e0
    return tau * delta if _kind_value(kind) == "pint-mqbvm" else delta


@dataclass(frozen=True)
class MethodSpec:
    """A method kind plus its regularisation parameter (methods.py:74-108)."""

    kind: MethodKind
    alpha: float

    def __post_init__(self):
        if not self.alpha > 0:
            raise ValueError(f"alpha must be positive, got {self.alpha}")

    def condition_divisor(self, tau: float) -> float:
        return condition_divisor(self.kind, self.alpha, tau)

    def omega(self, tau: float) -> Optional[float]:
        if not self.kind.is_circulant:
            return None
        return -tau / self.condition_divisor(tau)


def condition_divisor(kind, alpha: float, tau: float) -> float:
    """methods.py:85-96 -- tau*alpha (pint-qbvm), alpha (pint-mqbvm), 1 otherwise."""
    v = _kind_value(kind)
    if v == "pint-qbvm":
        return tau * alpha
    if v == "pint-mqbvm":
        return alpha
    return 1.0


class AllAtOnceSystem:
    """Stacked space-time system of a method for final data g (methods.py:111-171)."""

    def __init__(self, method: MethodSpec, grid: SpatialGrid, timegrid: TimeGrid, data):
        data = np.asarray(data, dtype=float)
        if data.shape != (grid.n_interior,):
            raise ValueError(f"final data must have shape ({grid.n_interior},), got {data.shape}")
        self.method = method
        self.grid = grid
        self.timegrid = timegrid
        self.data = data
        self.laplacian = LaplacianOperator(grid)

    @property
    def n_levels(self) -> int:
        return self.timegrid.n_levels

    @property
    def n_space(self) -> int:
        return self.grid.n_interior

    @property
    def size(self) -> int:
        return self.n_levels * self.n_space

    @property
    def omega(self) -> Optional[float]:
        return self.method.omega(self.timegrid.tau)

    def rhs(self) -> np.ndarray:
        """methods.py:158-162 -- scaled data in block 0, zeros elsewhere (host; the
        device solve never materialises it)."""
        out = np.zeros((self.n_levels, self.n_space))
        out[0] = self.data / self.method.condition_divisor(self.timegrid.tau)
        return out.ravel()

    def apply(self, states) -> np.ndarray:
        """Operator action (methods.py:164-171) for the pint kinds and the classic
        kinds (host numpy; residual checks only)."""
        states = np.asarray(states)
        flat = states.ndim == 1
        y = states.reshape(self.n_levels, self.n_space)
        tau = self.timegrid.tau
        alpha = self.method.alpha
        out = np.empty_like(y)
        out[1:] = (y[1:] - y[:-1]) / tau
        v = _kind_value(self.method.kind)
        if v == "qbvm":
            out[0] = alpha * y[0] + y[-1]
            out[1:] -= self.laplacian.apply(y[1:])
        elif v == "mqbvm":
            out[0] = (alpha / tau) * y[0] - (alpha / tau) * y[1] + y[-1]
            out[1:] -= self.laplacian.apply(y[1:])
        else:
            corner = 1.0 / self.method.condition_divisor(tau)
            out[0] = y[0] / tau + corner * y[-1]
            out -= self.laplacian.apply(y)
        return out.ravel() if flat else out


def assemble(kind, alpha: float, grid: SpatialGrid, timegrid: TimeGrid, data) -> AllAtOnceSystem:
    """methods.py:228-236."""
    return AllAtOnceSystem(MethodSpec(kind, alpha), grid, timegrid, data)


def residual(system, states) -> tuple:
    """methods.py:239-247 -- residual vector and its norm relative to the rhs."""
    rhs = system.rhs()
    vec = rhs - system.apply(np.asarray(states).ravel())
    return vec, float(np.linalg.norm(vec) / np.linalg.norm(rhs))


class SolveResult:
    """Outcome of one all-at-once solve (methods.py:250-285).

    ``trajectory`` is the (n_levels, n_space) float64 C-contiguous host array of
    the reference. The device solve keeps its output in HBM as
    ``trajectory_device`` (a torch tensor) and copies it to the host the first
    time ``trajectory`` is read, so callers that stay on the GPU never pay the
    device-to-host copy.
    """

    def __init__(self, system, trajectory, solver: str, timings: Optional[dict] = None, status: str = "ok",
                 message: str = "", trajectory_device=None):
        self.system = system
        self._trajectory = trajectory
        self.trajectory_device = trajectory_device
        self.solver = solver
        self.timings = dict(timings or {})
        self.status = status
        self.message = message

    @property
    def trajectory(self):
        if self._trajectory is None and self.trajectory_device is not None:
            self._trajectory = np.ascontiguousarray(self.trajectory_device.cpu().numpy())
        return self._trajectory

    @trajectory.setter
    def trajectory(self, value):
        self._trajectory = value

    @property
    def initial_state(self) -> np.ndarray:
        if self.trajectory is None:
            raise ValueError(f"no solution available (status={self.status!r})")
        return self.trajectory[0]

    @property
    def final_state(self) -> np.ndarray:
        if self.trajectory is None:
            raise ValueError(f"no solution available (status={self.status!r})")
        return self.trajectory[-1]

    def residual_norm(self) -> float:
        """Relative residual (methods.py:281-285). Device trajectories of the
        pint kinds are checked on the GPU (one fused stencil pass)."""
        if self._trajectory is None and self.trajectory_device is None:
            return float("nan")
        if self.trajectory_device is not None and self.system.method.kind.is_circulant:
            from .pint import device_residual_norm
            return device_residual_norm(self.system, self.trajectory_device)
        return residual(self.system, self.trajectory)[1]
