"""Dirichlet grids, the Laplacian spectrum, sine transforms and shifted solves.

Mirrors the reference module pkg/src/bhcp/space.py (same names, arguments,
return conventions and error types). Host code keeps the reference's exact
numpy expressions for the spectrum (space.py:209-215) so the device shifts
are bit-identical; the transforms and solves run on the B200 through
libbhcp_b200.so. Extension: ``dim`` may also be 3 (BASELINE config 4), with
the DST applied along axes -1, -2, -3 and the triple tensor sum spectrum.
"""

from __future__ import annotations

import functools
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from . import plans


class SingularShiftError(ArithmeticError):
    """A shifted operator s*I - lap is numerically singular for this grid (space.py:23-24)."""


@dataclass(frozen=True)
class SpatialGrid:
    """Uniform mesh on (0, L)^dim with homogeneous Dirichlet boundaries (space.py:27-74)."""

    dim: int
    length: float
    num_cells: int

    def __post_init__(self):
        if self.dim not in (1, 2, 3):
            raise ValueError(f"dim must be 1, 2 or 3, got {self.dim}")
        if not self.length > 0:
            raise ValueError(f"domain length must be positive, got {self.length}")
        if self.num_cells < 2:
            raise ValueError(f"need at least 2 cells per edge, got {self.num_cells}")

    @property
    def h(self) -> float:
        return self.length / self.num_cells

    @property
    def n_interior(self) -> int:
        return (self.num_cells - 1) ** self.dim

    @property
    def axis_nodes(self) -> np.ndarray:
        return self.h * np.arange(1, self.num_cells)

    def interior_coords(self) -> tuple:
        x = self.axis_nodes
        if self.dim == 1:
            return (x,)
        grids = np.meshgrid(*([x] * self.dim), indexing="ij")
        return tuple(g.ravel() for g in grids)


def build_grid(dim: int, length: float, num_cells: int) -> SpatialGrid:
    """space.py:77-79."""
    return SpatialGrid(dim=dim, length=length, num_cells=num_cells)


def grid_norm(values, grid: SpatialGrid) -> float:
    """Discrete L2 norm weighted by h**(dim/2) (space.py:82-89)."""
    values = np.asarray(values)
    if values.shape[-1] != grid.n_interior:
        raise ValueError(f"field has {values.shape[-1]} entries, grid has {grid.n_interior}")
    return float(grid.h ** (grid.dim / 2.0) * np.linalg.norm(values))


class LaplacianOperator:
    """Finite-difference Laplacian on interior nodes (space.py:92-127), host numpy.

    Used only for residual checks (methods.residual); the solve never applies it.
    """

    def __init__(self, grid: SpatialGrid):
        self.grid = grid

    def apply(self, values):
        grid = self.grid
        values = np.asarray(values)
        if values.shape[-1] != grid.n_interior:
            raise ValueError(f"field has {values.shape[-1]} entries, grid has {grid.n_interior}")
        inv_h2 = 1.0 / grid.h**2
        m = grid.num_cells - 1
        cube = values.reshape(values.shape[:-1] + (m,) * grid.dim)
        out = -2.0 * grid.dim * cube
        for ax in range(1, grid.dim + 1):
            lo = [slice(None)] * cube.ndim
            hi = [slice(None)] * cube.ndim
            lo[-ax] = slice(1, None)
            hi[-ax] = slice(None, -1)
            out[tuple(lo)] += cube[tuple(hi)]
            out[tuple(hi)] += cube[tuple(lo)]
        return (out * inv_h2).reshape(values.shape)

    __call__ = apply


def _sine_transform_device(grid: SpatialGrid, field):
    """Orthonormal DST-I along the trailing spatial axes on the device."""
    is_torch = isinstance(field, torch.Tensor)
    shape = tuple(field.shape)
    if shape[-1] != grid.n_interior:
        raise ValueError(f"field has {shape[-1]} entries, grid has {grid.n_interior}")
    cplx = torch.is_complex(field) if is_torch else np.iscomplexobj(field)
    dtype = torch.complex128 if cplx else torch.float64
    src = plans.to_device(field, dtype)
    batch = int(np.prod(shape[:-1], dtype=np.int64)) if len(shape) > 1 else 1
    out = torch.empty_like(src)
    sp = plan_for(grid)
    _lib.check(
        _lib.lib().bhcp_sine_transform(sp.handle, plans.ptr(src), plans.ptr(out), int(cplx), batch,
                                       plans.stream_handle()),
        "bhcp_sine_transform",
    )
    if is_torch:
        return out.reshape(shape)
    return out.reshape(shape).cpu().numpy()


@dataclass(frozen=True)
class SpatialSpectrum:
    """Sine-mode eigendecomposition of -lap (space.py:146-199)."""

    grid: SpatialGrid
    eigenvalues: np.ndarray
    mode_eigenvalues: np.ndarray

    def transform(self, field):
        return _sine_transform_device(self.grid, field)

    inverse = transform

    def mode(self, index) -> np.ndarray:
        m = self.grid.num_cells - 1
        j = np.arange(1, m + 1)
        idx = (index,) if self.grid.dim == 1 else tuple(index)
        if len(idx) != self.grid.dim:
            raise ValueError(f"mode index {index} does not match dim {self.grid.dim}")
        vecs = []
        for k in idx:
            k = int(k)
            if not 1 <= k <= m:
                raise ValueError(f"mode index {index} out of range 1..{m}")
            vecs.append(np.sqrt(2.0 / (m + 1)) * np.sin(k * j * np.pi / (m + 1)))
        out = vecs[0]
        for v in vecs[1:]:
            out = np.multiply.outer(out, v)
        return out.ravel()


def mu1_of(grid: SpatialGrid) -> np.ndarray:
    """space.py:209-211, verbatim expression."""
    k = np.arange(1, grid.num_cells)
    return (4.0 / grid.h**2) * np.sin(k * np.pi / (2.0 * grid.num_cells)) ** 2


@functools.lru_cache(maxsize=64)
def laplacian_eigenvalues(grid: SpatialGrid) -> SpatialSpectrum:
    """space.py:202-220 (3D: ((mu1 + mu1) + mu1) outer sum, same association)."""
    mu1 = mu1_of(grid)
    if grid.dim == 1:
        mode_mu = mu1
    elif grid.dim == 2:
        mode_mu = np.add.outer(mu1, mu1).ravel()
    else:
        mode_mu = np.add.outer(np.add.outer(mu1, mu1), mu1).ravel()
    return SpatialSpectrum(grid=grid, eigenvalues=np.sort(mode_mu), mode_eigenvalues=mode_mu)


def plan_for(grid: SpatialGrid) -> plans.SpacePlan:
    return plans.space_plan(grid.dim, grid.num_cells, mu1_of(grid))


def sine_transform(grid: SpatialGrid, field, direction: str = "forward"):
    """space.py:223-231 -- involutory orthonormal DST; direction only documents intent."""
    if direction not in ("forward", "inverse"):
        raise ValueError(f"direction must be 'forward' or 'inverse', got {direction!r}")
    return _sine_transform_device(grid, field)


def singular_message(shift) -> str:
    return (
        f"shift {shift} lies within 1e-14*|s| of an eigenvalue of the "
        f"Laplacian; the shifted operator is numerically singular"
    )


def solve_levels(grid: SpatialGrid, fields: torch.Tensor, shifts: np.ndarray) -> tuple:
    """Step (b) on level-major complex fields (levels, n_space) on the device.

    Returns (solution tensor, first singular column or -1). The singular-shift
    rule is evaluated inside the divide (space.py:237-240).
    """
    sp = plan_for(grid)
    sh = plans.to_device(np.ascontiguousarray(shifts, dtype=np.complex128), torch.complex128)
    status = plans.status_block()
    plans.reset_status(status)
    out = torch.empty_like(fields)
    _lib.check(
        _lib.lib().bhcp_step_b(sp.handle, plans.ptr(fields), plans.ptr(out), plans.ptr(sh), fields.shape[0],
                               plans.ptr(status), plans.stream_handle()),
        "bhcp_step_b",
    )
    st = plans.read_status(status)
    return out, int(st.bad_column)


def shifted_solve(grid: SpatialGrid, shift: complex, rhs, backend: str = "spectral"):
    """Solve (shift*I - lap) x = rhs (space.py:249-283).

    Both backends run the spectral device solve; ``"banded"`` is accepted for
    signature compatibility (the reference's LAPACK/SuperLU cross-check path,
    space.py:286-299, agrees with it to 1e-10 per test_space.py:176-186).
    """
    is_torch = isinstance(rhs, torch.Tensor)
    shape = tuple(rhs.shape) if is_torch else np.asarray(rhs).shape
    if shape != (grid.n_interior,):
        raise ValueError(f"rhs must have shape ({grid.n_interior},), got {shape}")
    if backend not in ("spectral", "banded"):
        raise ValueError(f"unknown backend {backend!r}")
    shift = complex(shift)
    rhs_cplx = torch.is_complex(rhs) if is_torch else np.iscomplexobj(rhs)
    real_data = shift.imag == 0.0 and not rhs_cplx
    fields = plans.to_device(rhs, torch.complex128).reshape(1, -1)
    out, bad = solve_levels(grid, fields, np.array([shift]))
    if bad >= 0:
        raise SingularShiftError(singular_message(shift))
    out = out.reshape(-1)
    if real_data:
        out = out.real.contiguous()
    return out if is_torch else out.cpu().numpy()
