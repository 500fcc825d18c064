"""Omega-circulant time coupling and its FFT diagonalisation (mirrors
pkg/src/bhcp/circulant.py).

``diagonalize`` keeps the reference's host numpy expressions (circulant.py:
143-153) so gamma and the eigenvalues are bit-identical; the transforms V and
V^{-1} (circulant.py:99-115) and the back rotation with its imaginary-residue
check (circulant.py:167-190) run on the B200 (k_time in libbhcp_b200.so).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from . import plans


class ImaginaryResidueError(ArithmeticError):
    """A nominally real result came back with a non-negligible imaginary part."""


@dataclass(frozen=True)
class TimeGrid:
    """Backward Euler partition of [0, horizon] into num_steps steps (circulant.py:28-58)."""

    horizon: float
    num_steps: int

    def __post_init__(self):
        if not self.horizon > 0:
            raise ValueError(f"time horizon must be positive, got {self.horizon}")
        if self.num_steps < 1:
            raise ValueError(f"need at least one time step, got {self.num_steps}")

    @property
    def tau(self) -> float:
        return self.horizon / self.num_steps

    @property
    def n_levels(self) -> int:
        return self.num_steps + 1

    @property
    def times(self) -> np.ndarray:
        return self.tau * np.arange(self.n_levels)


def step_matrix(size: int, omega: complex) -> np.ndarray:
    """Dense omega-circulant coupling, for tests and small cases (circulant.py:61-80)."""
    n = int(size)
    if n < 1:
        raise ValueError(f"matrix size must be at least 1, got {n}")
    if omega == 0:
        raise ValueError("omega must be nonzero")
    if n == 1:
        return np.array([[1.0 - omega]])
    mat = np.eye(n, dtype=np.result_type(omega, float))
    idx = np.arange(n - 1)
    mat[idx + 1, idx] = -1.0
    mat[0, n - 1] = -omega
    return mat


def _time_transform(block, diag, mode: int, tol: float | None = None, real_out: bool = False):
    """Run k_time along the trailing axis of ``block`` (numpy or torch).

    mode 0: ifft_ortho(block * gamma)  (apply_inverse_basis)
    mode 1: fft_ortho(block) / gamma   (apply_basis; real_out -> Re + residue)
    """
    is_torch = isinstance(block, torch.Tensor)
    shape = tuple(block.shape) if is_torch else np.asarray(block).shape
    n = diag.size
    if len(shape) == 0 or shape[-1] != n:
        raise ValueError(f"expected trailing axis {n}, got {shape[-1] if shape else None}")
    cplx_in = torch.is_complex(block) if is_torch else np.iscomplexobj(block)
    if mode == 1:
        cplx_in = True
    src = plans.to_device(block, torch.complex128 if cplx_in else torch.float64)
    batch = int(np.prod(shape[:-1], dtype=np.int64)) if len(shape) > 1 else 1
    tp = diag.plan()
    lib = _lib.lib()
    stream = plans.stream_handle()
    if mode == 0:
        out = torch.empty(shape, dtype=torch.complex128, device=src.device)
        _lib.check(
            lib.bhcp_to_eigenspace(tp.handle, plans.ptr(src), int(cplx_in), batch, n, 1, plans.ptr(out), n, 1,
                                   stream),
            "bhcp_to_eigenspace",
        )
        return out if is_torch else out.cpu().numpy()
    status = plans.status_block()
    plans.reset_status(status)
    out = torch.empty(shape, dtype=torch.float64 if real_out else torch.complex128, device=src.device)
    _lib.check(
        lib.bhcp_from_eigenspace(tp.handle, plans.ptr(src), batch, n, 1, plans.ptr(out), int(not real_out), n, 1,
                                 plans.ptr(status), stream),
        "bhcp_from_eigenspace",
    )
    if tol is not None:
        st = plans.read_status(status, tol)
        if st.code == _lib.BHCP_ERR_IMAGINARY_RESIDUE:
            raise ImaginaryResidueError(
                f"imaginary residue {st.residue:.3e} exceeds {tol:.1e} of the result norm {st.norm:.3e}"
            )
    return out if is_torch else out.cpu().numpy()


@dataclass(frozen=True)
class CirculantDiagonalization:
    """C = V diag(eigenvalues) V^{-1} of a step matrix (circulant.py:83-131)."""

    size: int
    omega: complex
    gamma: np.ndarray
    eigenvalues: np.ndarray

    def plan(self, tau: float | None = None) -> plans.TimePlan:
        shifts = self.eigenvalues / tau if tau is not None else self.eigenvalues
        return plans.time_plan(self.gamma, shifts)

    def apply_inverse_basis(self, values):
        """V^{-1} = F Gamma along the trailing axis (circulant.py:99-106)."""
        return _time_transform(values, self, 0)

    def apply_basis(self, coeffs):
        """V = Gamma^{-1} F^* along the trailing axis (circulant.py:108-115)."""
        return _time_transform(coeffs, self, 1)

    def basis_matrix(self) -> np.ndarray:
        return self.apply_basis(np.eye(self.size)).T

    def reconstruct(self) -> np.ndarray:
        return self.apply_basis(self.eigenvalues * self.apply_inverse_basis(np.eye(self.size))).T

    @property
    def condition_gamma(self) -> float:
        scale = max(abs(self.omega), 1.0 / abs(self.omega))
        return scale ** ((self.size - 1) / self.size)


def diagonalize(size: int, omega: complex) -> CirculantDiagonalization:
    """circulant.py:134-153 -- host numpy, identical expressions."""
    n = int(size)
    if n < 1:
        raise ValueError(f"matrix size must be at least 1, got {n}")
    omega = complex(omega)
    if omega == 0:
        raise ValueError("omega must be nonzero")
    gamma = np.exp(np.arange(n) * (np.log(omega) / n))
    root = gamma[1] if n > 1 else omega
    eigenvalues = 1.0 - root * np.exp(2j * np.pi * np.arange(n) / n)
    return CirculantDiagonalization(size=n, omega=omega, gamma=gamma, eigenvalues=eigenvalues)


def to_eigenspace(block, diag: CirculantDiagonalization):
    """Map a space-by-time block into the circulant eigenbasis (circulant.py:156-164)."""
    return diag.apply_inverse_basis(block)


def from_eigenspace(block, diag: CirculantDiagonalization, tol: float = 1e-8):
    """Back rotation, imaginary-residue check, real part (circulant.py:167-190)."""
    return _time_transform(block, diag, 1, tol=tol, real_out=True)
