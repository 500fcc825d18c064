"""numpy restatement of the reference PinT path -- TEST INFRASTRUCTURE ONLY.

See ``oracle/__init__.py``. Every function cites the reference line it
follows (``pkg/src/bhcp/<file>.py:<line>``). Third-party arithmetic used by the
reference and restated here through the same library calls:

* numpy.fft (pocketfft; numpy 2.3.5 in this image) -- circulant.py:106,115
* scipy.fft.dst type=1 norm="ortho" (pocketfft; scipy 1.18.1) -- space.py:172-176

``dst1_dense`` gives a library-independent DST-I (explicit sine matrix) so
the scipy call itself is pinned at small sizes.

Dimensions: the reference supports dim 1 and 2 (space.py:42-43). This
restatement extends every spatial routine to dim 3 by applying the same
1D operator along each axis (space.py:173-177 pattern) and the triple
tensor sum of the 1D spectrum (space.py:215 pattern). That extension is
"parity unpinned" against the reference proper and is pinned instead by
separable-mode reductions to the 1D/2D golden cases (tests/test_oracle.py).
"""

from __future__ import annotations

import numpy as np
import scipy.fft

PINT_QBVM = "pint-qbvm"
PINT_MQBVM = "pint-mqbvm"
QBVM = "qbvm"
MQBVM = "mqbvm"


# --------------------------------------------------------------------------
# time grid / method scalars
# --------------------------------------------------------------------------

def tau_of(horizon: float, num_steps: int) -> float:
    """circulant.py:45-48 -- tau = horizon / num_steps."""
    return horizon / num_steps


def condition_divisor(kind: str, alpha: float, tau: float) -> float:
    """methods.py:85-96 -- tau*alpha (pint-qbvm), alpha (pint-mqbvm), else 1."""
    if kind == PINT_QBVM:
        return tau * alpha
    if kind == PINT_MQBVM:
        return alpha
    return 1.0


def omega_of(kind: str, alpha: float, tau: float) -> float:
    """methods.py:98-108 -- omega = -tau / divisor for the circulant kinds."""
    if kind not in (PINT_QBVM, PINT_MQBVM):
        raise ValueError(f"{kind} has no circulant time coupling")
    return -tau / condition_divisor(kind, alpha, tau)


# --------------------------------------------------------------------------
# circulant diagonalisation and time transforms
# --------------------------------------------------------------------------

def diagonalize(n: int, omega: complex):
    """circulant.py:134-153 -- principal-branch gamma and eigenvalues d_j."""
    n = int(n)
    if n < 1:
        raise ValueError("size must be >= 1")
    omega = complex(omega)
    if omega == 0:
        raise ValueError("omega must be nonzero")
    gamma = np.exp(np.arange(n) * (np.log(omega) / n))
    root = gamma[1] if n > 1 else omega
    eig = 1.0 - root * np.exp(2j * np.pi * np.arange(n) / n)
    return gamma, eig


def condition_gamma(n: int, omega: complex) -> float:
    """circulant.py:127-131."""
    scale = max(abs(omega), 1.0 / abs(omega))
    return scale ** ((n - 1) / n)


def to_eigenspace(block, gamma):
    """circulant.py:99-106, 156-164 -- ifft_ortho(block * gamma) on the last axis."""
    block = np.asarray(block, dtype=np.complex128)
    if block.shape[-1] != gamma.shape[0]:
        raise ValueError("trailing axis mismatch")
    return np.fft.ifft(block * gamma, axis=-1, norm="ortho")


def apply_basis(coeffs, gamma):
    """circulant.py:108-115 -- fft_ortho(coeffs) / gamma on the last axis."""
    coeffs = np.asarray(coeffs, dtype=np.complex128)
    if coeffs.shape[-1] != gamma.shape[0]:
        raise ValueError("trailing axis mismatch")
    return np.fft.fft(coeffs, axis=-1, norm="ortho") / gamma


class ResidueError(ArithmeticError):
    pass


class SingularShift(ArithmeticError):
    pass


def from_eigenspace(block, gamma, tol=1e-8):
    """circulant.py:167-190 -- back rotation, residue check, real part."""
    out = apply_basis(block, gamma)
    scale = np.linalg.norm(out)
    residue = np.linalg.norm(out.imag)
    if residue > tol * max(scale, np.finfo(float).tiny):
        raise ResidueError(f"imaginary residue {residue:.3e} vs norm {scale:.3e}")
    return np.ascontiguousarray(out.real)


def residue_ratio(block, gamma) -> float:
    """||Im V x|| / ||V x|| of circulant.py:182-185, for reporting."""
    out = apply_basis(block, gamma)
    return float(np.linalg.norm(out.imag) / max(np.linalg.norm(out), np.finfo(float).tiny))


# --------------------------------------------------------------------------
# space: spectrum, DST-I, shifted solves (dim 1, 2 as reference; 3 restated)
# --------------------------------------------------------------------------

def mesh_width(length: float, num_cells: int) -> float:
    """space.py:49-52."""
    return length / num_cells


def mu1(length: float, num_cells: int) -> np.ndarray:
    """space.py:209-211 -- (4/h^2) sin^2(k pi / 2M), k = 1..M-1."""
    h = mesh_width(length, num_cells)
    k = np.arange(1, num_cells)
    return (4.0 / h**2) * np.sin(k * np.pi / (2.0 * num_cells)) ** 2


def mode_eigenvalues(dim: int, length: float, num_cells: int) -> np.ndarray:
    """space.py:212-215 -- tensor outer sum in C order (3D: triple sum)."""
    m1 = mu1(length, num_cells)
    if dim == 1:
        return m1
    if dim == 2:
        return np.add.outer(m1, m1).ravel()
    if dim == 3:
        return np.add.outer(np.add.outer(m1, m1), m1).ravel()
    raise ValueError(f"dim must be 1, 2 or 3, got {dim}")


def dst1_dense(m: int) -> np.ndarray:
    """Explicit orthonormal DST-I matrix, space.py:193 formula (sqrt(2/(m+1)) sin)."""
    j = np.arange(1, m + 1)
    return np.sqrt(2.0 / (m + 1)) * np.sin(np.outer(j, j) * np.pi / (m + 1))


def sine_transform(field, dim: int, m: int):
    """space.py:163-177 -- orthonormal DST-I along the trailing spatial axes.

    ``field`` has shape (..., m**dim). Axis order follows the reference:
    axis -1 first, then -2 (then -3 in the 3D restatement).
    """
    field = np.asarray(field)
    if field.shape[-1] != m**dim:
        raise ValueError("field size mismatch")
    if dim == 1:
        return scipy.fft.dst(field, type=1, norm="ortho", axis=-1)
    cube = field.reshape(field.shape[:-1] + (m,) * dim)
    out = cube
    for ax in range(1, dim + 1):
        out = scipy.fft.dst(out, type=1, norm="ortho", axis=-ax)
    return out.reshape(field.shape)


def check_shifts(shifts, mode_mu):
    """space.py:234-246 -- singular if min_k |s + mu_k| <= 1e-14 |s|; returns first bad index or -1."""
    shifts = np.atleast_1d(shifts)
    denom_min = np.min(np.abs(shifts[:, None] + mode_mu[None, :]), axis=1)
    bad = denom_min <= 1e-14 * np.abs(shifts)
    return int(np.argmax(bad)) if np.any(bad) else -1


def shifted_solve(shift, rhs, dim, length, num_cells):
    """space.py:249-283 (spectral backend) -- DST, divide by (s + mu), DST."""
    m = num_cells - 1
    mu = mode_eigenvalues(dim, length, num_cells)
    shift = complex(shift)
    if check_shifts(np.array([shift]), mu) >= 0:
        raise SingularShift(f"shift {shift} is singular")
    rhs = np.asarray(rhs)
    real_data = shift.imag == 0.0 and not np.iscomplexobj(rhs)
    coeffs = sine_transform(rhs.astype(np.complex128), dim, m)
    out = sine_transform(coeffs / (shift + mu), dim, m)
    return out.real if real_data else out


def step_b(block, shifts, dim, length, num_cells):
    """pint.py:26-66 -- one shifted solve per column j of an (n_space, n_levels) block."""
    block = np.asarray(block)
    shifts = np.atleast_1d(shifts)
    if block.ndim != 2 or block.shape[1] != shifts.shape[0]:
        raise ValueError("need one shift per column")
    out = np.empty(block.shape, dtype=np.complex128)
    for j in range(shifts.shape[0]):
        try:
            out[:, j] = shifted_solve(shifts[j], block[:, j], dim, length, num_cells)
        except SingularShift as exc:
            raise SingularShift(f"column {j}: {exc}") from exc
    return out


# --------------------------------------------------------------------------
# all-at-once system pieces and solvers
# --------------------------------------------------------------------------

def rhs_block(data, kind, alpha, tau, n_levels):
    """methods.py:158-162 -- zeros with row 0 = data / divisor, shape (n_levels, n_space)."""
    data = np.asarray(data, dtype=float)
    out = np.zeros((n_levels, data.shape[0]))
    out[0] = data / condition_divisor(kind, alpha, tau)
    return out


def solve_pint(kind, alpha, dim, length, num_cells, horizon, num_steps, data):
    """pint.py:69-110 -- the reference 3-step solve, returns (trajectory, residue_ratio).

    trajectory is (n_levels, n_space) float64 C-contiguous, like pint.py:99.
    """
    tau = tau_of(horizon, num_steps)
    n = num_steps + 1
    gamma, eig = diagonalize(n, omega_of(kind, alpha, tau))
    rhs = rhs_block(data, kind, alpha, tau, n)
    s1 = to_eigenspace(rhs.T, gamma)
    s2 = step_b(s1, eig / tau, dim, length, num_cells)
    ratio = residue_ratio(s2, gamma)
    traj = np.ascontiguousarray(from_eigenspace(s2, gamma).T)
    return traj, ratio


def spectral_denominator(kind, alpha, tau, num_steps, mu):
    """baseline.py:90-99 -- (rho, per-mode denominator D_k)."""
    rho = 1.0 / (1.0 + tau * mu)
    decay = rho**num_steps
    if kind == QBVM:
        denom = alpha + decay
    elif kind == MQBVM:
        denom = alpha * mu * rho + decay
    elif kind == PINT_QBVM:
        denom = alpha * (1.0 + tau * mu) + decay
    else:
        denom = alpha * (mu + 1.0 / tau) + decay
    return rho, denom


def spectral_oracle(kind, alpha, dim, length, num_cells, horizon, num_steps, data,
                    levels=None):
    """baseline.py:67-112 -- closed-form per-mode solve (dim 3 by restatement).

    ``levels`` optionally restricts the returned rows (for sampled full-size
    checks); default is every level 0..N.
    """
    data = np.asarray(data, dtype=float)
    m = num_cells - 1
    mu = mode_eigenvalues(dim, length, num_cells)
    tau = tau_of(horizon, num_steps)
    rho, denom = spectral_denominator(kind, alpha, tau, num_steps, mu)
    amplitudes = sine_transform(data, dim, m) / denom
    if levels is None:
        levels = np.arange(num_steps + 1)
    levels = np.asarray(levels)
    return sine_transform(amplitudes[None, :] * rho[None, :] ** levels[:, None], dim, m)


def march_forward_spectral(z0, dim, length, num_cells, horizon, num_steps):
    """baseline.py:115-129 in its per-mode form: g = DST(rho^N DST(z0)).

    Equal to the N sequential shifted solves to roundoff (test_baseline.py:157-164).
    """
    m = num_cells - 1
    mu = mode_eigenvalues(dim, length, num_cells)
    tau = tau_of(horizon, num_steps)
    rho = 1.0 / (1.0 + tau * mu)
    return sine_transform(sine_transform(np.asarray(z0, float), dim, m) * rho**num_steps, dim, m)


def march_forward(z0, dim, length, num_cells, horizon, num_steps):
    """baseline.py:115-129 -- literal N-step recursion (small sizes only)."""
    state = np.asarray(z0, dtype=float)
    inv_tau = 1.0 / tau_of(horizon, num_steps)
    for _ in range(num_steps):
        state = shifted_solve(inv_tau, state * inv_tau, dim, length, num_cells)
    return state


def l2_error(reconstructed, exact, h, dim):
    """bench.py:154-162 -- sqrt(h^dim) * ||y - z||."""
    return float(np.sqrt(h**dim) * np.linalg.norm(np.asarray(reconstructed) - np.asarray(exact)))


def rel_l2(a, b) -> float:
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


def parity_tolerance(n_levels: int, omega: float) -> float:
    """max(1e-10, 10 * cond(Gamma) * DBL_EPSILON)."""
    return max(1e-10, 10.0 * condition_gamma(n_levels, omega) * np.finfo(float).eps)


# --------------------------------------------------------------------------
# bounded CPU-baseline sample (bench.py cpu_baseline / --impl reference)
# --------------------------------------------------------------------------

def solve_pint_sample(kind, alpha, dim, length, num_cells, horizon, num_steps, data,
                      fraction: float, workers=None):
    """Time the reference 3-step solve (pint.py:89-99) on a bounded sample.

    The sample performs a fraction ``f`` of every per-unit operation of the
    full solve, with the reference's own memory layouts:

    * step (a): the rhs rows (methods.py:158-162) and the time transforms of
      ceil(f*N_x) spatial rows (circulant.py:99-106);
    * step (b): ceil(f*N_t) columns j, each read as a strided column of the
      (N_x, cols) S1 block and written back as one (pint.py:52-61), each with
      the per-column singular-shift scan (space.py:234-246, 273) and the
      spectral solve (space.py:276-278); a ThreadPoolExecutor of ``workers``
      threads exactly like the reference's optional pool (pint.py:62-65);
    * step (c): the back transform of ceil(f*N_x) rows, both residue norms,
      the real part (circulant.py:108-115, 182-190) and the transposed
      contiguous copy of the trajectory rows (pint.py:99).

    Every operation is linear in the number of rows or columns it touches, so
    the full-solve time is extrapolated as elapsed / f. Returns
    (dof_equivalent, seconds) with dof_equivalent = f * N_t * N_x.
    """
    import time
    from concurrent.futures import ThreadPoolExecutor

    tau = tau_of(horizon, num_steps)
    n = num_steps + 1
    gamma, eig = diagonalize(n, omega_of(kind, alpha, tau))
    shifts = eig / tau
    data = np.asarray(data, dtype=float)
    nx = data.shape[0]
    m = num_cells - 1
    mu = mode_eigenvalues(dim, length, num_cells)
    rows = max(1, int(np.ceil(fraction * nx)))
    cols = max(1, int(np.ceil(fraction * n)))
    # S1 columns: column j of S1 is rhs_0 / sqrt(n) (the exact step-(a) output;
    # the values do not change the work)
    col = (data / condition_divisor(kind, alpha, tau) / np.sqrt(n)).astype(np.complex128)
    s1 = np.empty((nx, cols), dtype=np.complex128)
    s1[:] = col[:, None]
    start = time.perf_counter()
    # (a) rhs block rows (methods.py:158-162) and their time transform
    rhs_rows = np.zeros((rows, n))
    rhs_rows[:, 0] = data[:rows] / condition_divisor(kind, alpha, tau)
    s1_rows = to_eigenspace(rhs_rows, gamma)

    def solve_column(j):
        if check_shifts(np.array([shifts[j]]), mu) >= 0:
            raise SingularShift(f"column {j}")
        coeffs = sine_transform(s1[:, j], dim, m)
        return sine_transform(coeffs / (shifts[j] + mu), dim, m)

    out = np.empty((nx, cols), dtype=np.complex128)
    if workers is None:
        for j in range(cols):
            out[:, j] = solve_column(j)
    else:
        with ThreadPoolExecutor(max_workers=workers) as pool:
            for j, c in enumerate(pool.map(solve_column, range(cols))):
                out[:, j] = c
    # (c) back transform of sample rows + residue norms + real part + transposed copy
    back = apply_basis(s1_rows, gamma)
    _ = np.linalg.norm(back), np.linalg.norm(back.imag)
    _ = np.ascontiguousarray(np.ascontiguousarray(back.real).T)
    elapsed = time.perf_counter() - start
    return fraction * n * nx, elapsed


# --------------------------------------------------------------------------
# numpy restatement of the device's fused halves (tests of the multi-rank
# orchestration on CPU; see paper_2107_06381_b200/pint.py docstring)
# --------------------------------------------------------------------------

def fused_pass_a(kind, alpha, dim, length, num_cells, horizon, num_steps, data, k_begin, k_end):
    """W[t, k] = ghat_k / (divisor n) * Re(gamma_inv_t * FFT_j(1 / (s_j + mu_k)))
    for modes [k_begin, k_end); returns (W (n, S), sum Re^2, sum Im^2)."""
    tau = tau_of(horizon, num_steps)
    n = num_steps + 1
    gamma, eig = diagonalize(n, omega_of(kind, alpha, tau))
    shifts = eig / tau
    m = num_cells - 1
    mu = mode_eigenvalues(dim, length, num_cells)[k_begin:k_end]
    ghat = sine_transform(np.asarray(data, float), dim, m)[k_begin:k_end]
    c = ghat / (condition_divisor(kind, alpha, tau) * n)
    X = np.fft.fft(1.0 / (shifts[:, None] + mu[None, :]), axis=0)
    Z = X * (1.0 / gamma)[:, None] * c[None, :]
    return np.ascontiguousarray(Z.real), float(np.sum(Z.real**2)), float(np.sum(Z.imag**2))


def fused_pass_b(W_full_levels, dim, m):
    """Inverse DST of level-major real fields (L, m**dim)."""
    return sine_transform(W_full_levels, dim, m)
