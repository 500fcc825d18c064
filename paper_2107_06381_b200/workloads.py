"""Seeded synthetic inputs for the five BASELINE.json configurations.

No public dataset is involved: each config is restated on the reference API
(SURVEY.md section 8(d)). Seed convention: one ``numpy.random.default_rng(seed)``
per config; draw the z0 coefficients first, then the noise vector eps.

* z0 is sampled at interior nodes (space.py:60-74 ordering, first axis outermost).
* g is the discrete forward solve of z0 to t = T. The reference computes it
  with N sequential shifted solves (baseline.py:115-129); here the identical
  per-mode form g = DST(rho^N DST(z0)) is used (equal to roundoff, pinned by
  tests/test_workloads.py against the reference's own march_forward output).
* g_delta = g + delta * eps / ||eps|| * ||g||  (relative Gaussian noise).

Host-side input preparation only (numpy / scipy.fft); the solve itself never
runs here.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.fft


@dataclass
class Workload:
    name: str
    dim: int
    length: float
    num_cells: int
    horizon: float
    num_steps: int
    kinds: tuple
    alphas: tuple
    delta: float
    seed: int
    z0: np.ndarray = field(repr=False)
    g: np.ndarray = field(repr=False)
    g_delta: np.ndarray = field(repr=False)

    @property
    def n_levels(self) -> int:
        return self.num_steps + 1

    @property
    def n_space(self) -> int:
        return (self.num_cells - 1) ** self.dim

    @property
    def dof(self) -> int:
        return self.n_levels * self.n_space

    @property
    def h(self) -> float:
        return self.length / self.num_cells

    @property
    def tau(self) -> float:
        return self.horizon / self.num_steps


CONFIGS = {
    # name: (dim, length, M, T, N, kinds, alphas, delta, kmax)
    "c1": (1, np.pi, 256, 1.0, 256, ("pint-qbvm",), (1e-3,), 1e-3, 8),
    "c2": (2, 1.0, 512, 0.1, 512, ("pint-mqbvm",), (1e-2,), 1e-2, 16),
    "c3": (2, 1.0, 1024, 0.1, 1024, ("pint-qbvm",), (1e-3,), 1e-3, 16),
    "c4": (3, 1.0, 256, 0.05, 256, ("pint-mqbvm",), (1e-2,), 1e-2, 8),
    "c5": (1, np.pi, 4096, 1.0, 4096, ("pint-qbvm", "pint-mqbvm"), tuple(np.logspace(-6, -1, 64)), 1e-4, 8),
}
SEEDS = {"c1": 1, "c2": 2, "c3": 3, "c4": 4, "c5": 5}


def dst_all_axes(x: np.ndarray, dim: int, m: int) -> np.ndarray:
    cube = x.reshape((m,) * dim)
    for ax in range(1, dim + 1):
        cube = scipy.fft.dst(cube, type=1, norm="ortho", axis=-ax)
    return cube.reshape(-1)


def mu_modes(dim: int, length: float, num_cells: int) -> np.ndarray:
    h = length / num_cells
    k = np.arange(1, num_cells)
    mu1 = (4.0 / h**2) * np.sin(k * np.pi / (2.0 * num_cells)) ** 2
    out = mu1
    for _ in range(dim - 1):
        out = np.add.outer(out, mu1)
    return out.ravel()


def initial_state(rng, dim: int, length: float, num_cells: int, kmax: int) -> np.ndarray:
    """z0 = sum c_k prod_a sin(k_a pi x_a / length) with c ~ N(0,1)/|k|^2."""
    h = length / num_cells
    x = h * np.arange(1, num_cells)
    ks = np.arange(1, kmax + 1)
    if dim == 1:
        coef = rng.standard_normal(kmax) / ks**2
        # length pi: sin(k x); length 1: sin(k pi x) -- both are sin(k pi x / length)
        return np.sin(np.outer(x, ks) * (np.pi / length)) @ coef
    grids = np.meshgrid(*([ks] * dim), indexing="ij")
    ksq = sum(g.astype(float) ** 2 for g in grids)
    coef = rng.standard_normal((kmax,) * dim) / ksq
    S = np.sin(np.outer(x, ks) * (np.pi / length))  # (m, kmax)
    if dim == 2:
        return (S @ coef @ S.T).ravel()
    return np.einsum("ia,jb,kc,abc->ijk", S, S, S, coef, optimize=True).ravel()


def forward_data(z0: np.ndarray, dim: int, length: float, num_cells: int, horizon: float, num_steps: int):
    """g = DST(rho^N DST(z0)) -- march_forward (baseline.py:115-129) in per-mode form."""
    m = num_cells - 1
    tau = horizon / num_steps
    rho = 1.0 / (1.0 + tau * mu_modes(dim, length, num_cells))
    return dst_all_axes(dst_all_axes(z0, dim, m) * rho**num_steps, dim, m)


def make(name: str, seed: int | None = None) -> Workload:
    dim, length, M, T, N, kinds, alphas, delta, kmax = CONFIGS[name]
    seed = SEEDS[name] if seed is None else seed
    rng = np.random.default_rng(seed)
    z0 = initial_state(rng, dim, length, M, kmax)
    g = forward_data(z0, dim, length, M, T, N)
    eps = rng.standard_normal(g.shape[0])
    g_delta = g + delta * eps / np.linalg.norm(eps) * np.linalg.norm(g)
    return Workload(name, dim, length, M, T, N, kinds, alphas, delta, seed, z0, g, g_delta)


def make_small(dim: int, num_cells: int, num_steps: int, seed: int = 7, length: float = 1.0,
               horizon: float = 0.1, delta: float = 1e-2, kmax: int = 4) -> Workload:
    """Same construction at a reduced size (parity tests)."""
    rng = np.random.default_rng(seed)
    z0 = initial_state(rng, dim, length, num_cells, min(kmax, num_cells - 1))
    g = forward_data(z0, dim, length, num_cells, horizon, num_steps)
    eps = rng.standard_normal(g.shape[0])
    g_delta = g + delta * eps / np.linalg.norm(eps) * np.linalg.norm(g)
    return Workload(f"small{dim}d", dim, length, num_cells, horizon, num_steps, ("pint-qbvm", "pint-mqbvm"),
                    (delta,), delta, seed, z0, g, g_delta)


def l2_error(reconstructed, exact, h: float, dim: int) -> float:
    """bench.py:154-162 -- sqrt(h**dim) * ||y - z||."""
    reconstructed = np.asarray(reconstructed)
    exact = np.asarray(exact)
    if reconstructed.shape != exact.shape:
        raise ValueError(f"shape mismatch: {reconstructed.shape} vs {exact.shape}")
    return float(np.sqrt(h**dim) * np.linalg.norm(reconstructed - exact))
