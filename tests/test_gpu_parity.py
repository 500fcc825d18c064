"""Device parity: every CUDA entry point against the CPU oracle / the
reference's golden vectors on the same seeded inputs (B200 only).

Tolerances: the north-star bar is relative L2 <= 1e-10 in fp64; where the
reference's own result is conditioned by Gamma (cond(Gamma) up to 1e6) the bar
is max(1e-10, 10 * cond(Gamma) * eps) (oracle.parity_tolerance).
Transform-level checks use the tighter per-transform bars stated inline.
"""

import numpy as np
import pytest
import torch

import paper_2107_06381_b200 as B
from oracle import bhcp_oracle as O
from paper_2107_06381_b200 import workloads

pytestmark = pytest.mark.gpu


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


# ----------------------------------------------------------------- transforms

@pytest.mark.parametrize("dim,cells", [(1, 2), (1, 8), (1, 16), (1, 33), (2, 3), (2, 7), (2, 8)])
def test_sine_transform_golden(golden, dim, cells):
    grid = B.build_grid(dim, np.pi, cells)
    key = f"{dim}_{cells}"
    assert rel(B.sine_transform(grid, golden[f"dst_real_in_{key}"]), golden[f"dst_real_out_{key}"]) <= 1e-14
    out = B.sine_transform(grid, golden[f"dst_cplx_in_{key}"])
    assert np.iscomplexobj(out)
    assert rel(out, golden[f"dst_cplx_out_{key}"]) <= 1e-14


@pytest.mark.parametrize("cells", list(range(2, 70)) + [128, 255, 256, 257, 512, 1024, 2048, 4096])
def test_sine_transform_lengths_1d(cells):
    rng = np.random.default_rng(cells)
    m = cells - 1
    x = rng.standard_normal((3, m))
    grid = B.build_grid(1, 1.0, cells)
    assert rel(B.sine_transform(grid, x), O.sine_transform(x, 1, m)) <= 1e-14
    z = x + 1j * rng.standard_normal((3, m))
    assert rel(B.sine_transform(grid, z), O.sine_transform(z, 1, m)) <= 1e-14


@pytest.mark.parametrize("dim,cells,batch", [(2, 5, 3), (2, 16, 2), (2, 33, 1), (3, 5, 2), (3, 9, 1), (3, 17, 1)])
def test_sine_transform_multi_d(dim, cells, batch):
    rng = np.random.default_rng(dim * 100 + cells)
    m = cells - 1
    x = rng.standard_normal((batch, m**dim))
    grid = B.build_grid(dim, 1.0, cells)
    assert rel(B.sine_transform(grid, x), O.sine_transform(x, dim, m)) <= 1e-14
    z = x + 1j * rng.standard_normal(x.shape)
    assert rel(B.sine_transform(grid, z), O.sine_transform(z, dim, m)) <= 1e-14


def test_sine_transform_involutory_and_direction():
    grid = B.build_grid(2, np.pi, 7)
    x = np.random.default_rng(11).standard_normal(36)
    back = B.sine_transform(grid, B.sine_transform(grid, x), "inverse")
    assert np.allclose(back, x, atol=1e-12)
    with pytest.raises(ValueError):
        B.sine_transform(grid, x, "sideways")


@pytest.mark.parametrize("n", [2, 3, 4, 5, 8, 9, 17, 33, 65, 257, 513])
def test_time_transforms_golden(golden, n):
    d = B.diagonalize(n, complex(golden[f"toeig_omega_{n}"]))
    s = B.to_eigenspace(golden[f"toeig_in_{n}"], d)
    assert rel(s, golden[f"toeig_out_{n}"]) <= 1e-14
    back = B.from_eigenspace(golden[f"toeig_out_{n}"], d)
    assert back.dtype == np.float64 and back.flags["C_CONTIGUOUS"]
    assert rel(back, golden[f"fromeig_out_{n}"]) <= 1e-12 * d.condition_gamma


@pytest.mark.parametrize("n", list(range(1, 70)) + [127, 241, 257, 481, 513, 1025, 2049, 4097])
def test_time_transform_lengths(n):
    rng = np.random.default_rng(n)
    blk = rng.standard_normal((4, n)) + 1j * rng.standard_normal((4, n))
    d = B.diagonalize(n, -3.0)
    assert rel(B.to_eigenspace(blk, d), O.to_eigenspace(blk, d.gamma)) <= 2e-15 * max(1, np.log2(n))
    assert rel(d.apply_basis(blk), O.apply_basis(blk, d.gamma)) <= 2e-15 * max(1, np.log2(n)) * d.condition_gamma


def test_omega_one_is_plain_dft():
    d = B.diagonalize(8, 1.0)
    blk = np.random.default_rng(13).standard_normal((3, 8))
    assert np.allclose(B.to_eigenspace(blk, d), np.fft.ifft(blk, axis=-1, norm="ortho"), atol=1e-13)


def test_round_trip_and_residue_error():
    for omega in (-1e4, -1.0, -1e-4, 2.0):
        d = B.diagonalize(8, omega)
        blk = np.random.default_rng(21).standard_normal((5, 8))
        back = B.from_eigenspace(B.to_eigenspace(blk, d), d)
        assert np.linalg.norm(back - blk) <= 1e-10 * max(abs(omega), 1 / abs(omega)) * np.linalg.norm(blk)
    d = B.diagonalize(8, 2.0)
    rng = np.random.default_rng(31)
    garbage = rng.standard_normal((2, 8)) + 1j * rng.standard_normal((2, 8))
    with pytest.raises(B.ImaginaryResidueError):
        B.from_eigenspace(garbage, d)
    with pytest.raises(ValueError):
        B.to_eigenspace(np.zeros((3, 7)), d)


def test_reconstruction_within_conditioning():
    for size in (2, 3, 4, 8, 16):
        for omega in (-1e4, -1.0, -1e-4, 2.0):
            d = B.diagonalize(size, omega)
            target = B.step_matrix(size, omega)
            err = np.linalg.norm(d.reconstruct() - target)
            assert err <= 1e-10 * d.condition_gamma * np.linalg.norm(target)


# ----------------------------------------------------------------- step (b)

@pytest.mark.parametrize("dim,cells", [(1, 16), (2, 8)])
def test_shifted_solve_golden(golden, dim, cells):
    grid = B.build_grid(dim, np.pi, cells)
    rhs = golden[f"ssolve_rhs_{dim}_{cells}"]
    for i in range(3):
        s = complex(golden[f"ssolve_shift_{dim}_{cells}_{i}"])
        for backend in ("spectral", "banded"):
            out = B.shifted_solve(grid, s, rhs, backend=backend)
            assert rel(out, golden[f"ssolve_out_{dim}_{cells}_{i}"]) <= 1e-13


def test_shifted_solve_3d_vs_oracle():
    rng = np.random.default_rng(5)
    grid = B.build_grid(3, 1.0, 7)
    rhs = rng.standard_normal(216) + 1j * rng.standard_normal(216)
    for s in (4.0, 3.0 + 2.0j, -0.5 + 40.0j):
        assert rel(B.shifted_solve(grid, s, rhs), O.shifted_solve(s, rhs, 3, 1.0, 7)) <= 1e-13


def test_shifted_solve_semantics():
    grid = B.build_grid(1, np.pi, 8)
    assert np.array_equal(B.shifted_solve(grid, 1.5, np.zeros(7)), np.zeros(7))
    assert not np.iscomplexobj(B.shifted_solve(grid, 2.0, np.ones(7)))
    assert np.iscomplexobj(B.shifted_solve(grid, 2.0 + 1.0j, np.ones(7)))
    mu1 = B.laplacian_eigenvalues(grid).eigenvalues[0]
    with pytest.raises(B.SingularShiftError):
        B.shifted_solve(grid, -mu1, np.ones(7))
    with pytest.raises(ValueError):
        B.shifted_solve(grid, 1.0, np.ones(6))
    with pytest.raises(ValueError):
        B.shifted_solve(grid, 1.0, np.ones(7), backend="cholesky")


def test_shifted_solve_residual_2d():
    grid = B.build_grid(2, np.pi, 6)
    lap = B.LaplacianOperator(grid)
    rhs = np.random.default_rng(29).standard_normal(grid.n_interior)
    x = B.shifted_solve(grid, 7.0, rhs)
    assert np.linalg.norm(7.0 * x - lap.apply(x) - rhs) <= 1e-12 * np.linalg.norm(rhs)


def test_step_b_golden_and_errors(golden):
    grid = B.build_grid(1, np.pi, 16)
    out = B.step_b_parallel(grid, golden["stepb_in"], golden["stepb_shifts"])
    assert rel(out, golden["stepb_out"]) <= 1e-13
    again = B.step_b_parallel(grid, golden["stepb_in"], golden["stepb_shifts"], workers=3)
    assert np.array_equal(out, again)
    g8 = B.build_grid(1, np.pi, 8)
    mu1 = B.laplacian_eigenvalues(g8).eigenvalues[0]
    with pytest.raises(B.SingularShiftError, match="column 2"):
        B.step_b_parallel(g8, np.ones((7, 4), dtype=complex), np.array([1.0, 2.0, -mu1, 4.0]))
    with pytest.raises(ValueError):
        B.step_b_parallel(g8, np.ones((7, 3)), np.ones(4))


def test_step_b_sine_mode_closed_form():
    grid = B.build_grid(1, np.pi, 8)
    spectrum = B.laplacian_eigenvalues(grid)
    diag = B.diagonalize(9, -4.0)
    shifts = diag.eigenvalues / 0.125
    mode = spectrum.mode(3)
    out = B.step_b_parallel(grid, np.tile(mode[:, None], (1, 9)).astype(complex), shifts)
    expected = mode[:, None] / (shifts[None, :] + spectrum.eigenvalues[2])
    assert np.allclose(out, expected, atol=1e-13)


# ----------------------------------------------------------------- full solve

CASES = ["1d_m8_n8", "1d_m16_n16", "1d_m4_n4", "2d_m6_n5", "2d_m8_n8"]


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("kind", [B.MethodKind.PINT_QBVM, B.MethodKind.PINT_MQBVM])
def test_solve_pint_golden(golden, name, kind):
    dim, length, cells, horizon, steps, alpha = golden[f"case_{name}_params"]
    grid = B.build_grid(int(dim), length, int(cells))
    system = B.assemble(kind, alpha, grid, B.TimeGrid(horizon, int(steps)), golden[f"case_{name}_data"])
    res = B.solve_pint(system)
    y = res.trajectory
    assert y.shape == (system.n_levels, system.n_space) and y.dtype == np.float64 and y.flags["C_CONTIGUOUS"]
    oracle = golden[f"oracle_{name}_{kind.value}"]
    tol = O.parity_tolerance(system.n_levels, system.omega)
    assert rel(y, oracle) <= tol
    assert rel(y, golden[f"pint_{name}_{kind.value}"]) <= tol
    unf = B.solve_pint_unfused(system).trajectory
    assert rel(unf, oracle) <= tol


def test_solve_pint_c1_golden(golden):
    grid = B.build_grid(1, np.pi, 256)
    tg = B.TimeGrid(1.0, 256)
    system = B.assemble(B.MethodKind.PINT_QBVM, 1e-3, grid, tg, golden["c1_gdelta"])
    res = B.solve_pint(system)
    assert rel(res.trajectory, golden["c1_oracle"]) <= 1e-10
    assert rel(res.trajectory, golden["c1_pint"]) <= 1e-10
    e_gpu = workloads.l2_error(res.initial_state, golden["c1_z0"], grid.h, 1)
    e_orc = workloads.l2_error(golden["c1_oracle"][0], golden["c1_z0"], grid.h, 1)
    assert abs(e_gpu - e_orc) <= 5e-4 * abs(e_orc)  # 3 significant digits
    t = res.timings
    assert set(t) >= {"step_a", "step_b", "step_c", "total"}
    assert t["total"] == pytest.approx(t["step_a"] + t["step_b"] + t["step_c"], abs=1e-9)


def test_result_semantics():
    grid = B.build_grid(1, np.pi, 8)
    zero = B.assemble(B.MethodKind.PINT_QBVM, 0.1, grid, B.TimeGrid(1.0, 8), np.zeros(7))
    assert not B.solve_pint(zero).trajectory.any()
    data = np.random.default_rng(4).standard_normal(7)
    system = B.assemble(B.MethodKind.PINT_QBVM, 1e-3, grid, B.TimeGrid(1.0, 8), data)
    r1 = B.solve_pint(system)
    r2 = B.solve_pint(system, workers=4)
    assert np.array_equal(r1.trajectory, r2.trajectory)
    assert np.array_equal(r1.initial_state, r1.trajectory[0])
    assert np.array_equal(r1.final_state, r1.trajectory[-1])
    assert r1.residual_norm() <= 1e-8 * max(1.0, abs(system.omega))
    assert r1.solver == "pint" and r1.status == "ok"


@pytest.mark.parametrize("dim,cells,steps", [(1, 64, 63), (1, 100, 40), (2, 16, 16), (2, 20, 33), (3, 8, 8),
                                             (3, 12, 10),
                                             # the specialised pass-A kernels: n = 257 (Rader), 513 (Stockham),
                                             # 1025 (Good-Thomas + Rader), 4097 (prime factor + Rader); 2D / 3D
                                             # run their symmetric (mirror / permutation-class) tile lists
                                             (1, 32, 256), (2, 12, 256), (3, 6, 256), (2, 10, 512), (2, 8, 1024),
                                             (3, 5, 1024), (1, 16, 4096), (2, 6, 4096), (3, 4, 4096)])
@pytest.mark.parametrize("alpha", [1e-1, 1e-3, 1e-6])
def test_solve_pint_sizes_vs_oracle(dim, cells, steps, alpha):
    w = workloads.make_small(dim, cells, steps, seed=cells + steps)
    grid = B.build_grid(dim, w.length, cells)
    tg = B.TimeGrid(w.horizon, steps)
    for kind in (B.MethodKind.PINT_QBVM, B.MethodKind.PINT_MQBVM):
        system = B.assemble(kind, alpha, grid, tg, w.g_delta)
        y = B.solve_pint(system).trajectory
        ref = O.spectral_oracle(kind.value, alpha, dim, w.length, cells, w.horizon, steps, w.g_delta)
        assert rel(y, ref) <= O.parity_tolerance(tg.n_levels, system.omega)


def test_c2_full_size_vs_oracle():
    """BASELINE config 2 at full size: rel-L2 over the whole trajectory and e_h."""
    w = workloads.make("c2")
    grid = B.build_grid(2, w.length, w.num_cells)
    tg = B.TimeGrid(w.horizon, w.num_steps)
    system = B.assemble(B.MethodKind.PINT_MQBVM, 1e-2, grid, tg, w.g_delta)
    res = B.solve_pint(system)
    y = res.trajectory
    ref = O.spectral_oracle("pint-mqbvm", 1e-2, 2, w.length, w.num_cells, w.horizon, w.num_steps, w.g_delta)
    assert rel(y, ref) <= 1e-10
    e_gpu = workloads.l2_error(y[0], w.z0, grid.h, 2)
    e_orc = workloads.l2_error(ref[0], w.z0, grid.h, 2)
    assert abs(e_gpu - e_orc) <= 5e-4 * abs(e_orc)


@pytest.mark.parametrize("alpha_idx", [0, 21, 42, 63])
def test_c5_sweep_samples_vs_oracle(alpha_idx):
    w = workloads.make("c5")
    alpha = w.alphas[alpha_idx]
    grid = B.build_grid(1, w.length, w.num_cells)
    tg = B.TimeGrid(w.horizon, w.num_steps)
    for kind in (B.MethodKind.PINT_QBVM, B.MethodKind.PINT_MQBVM):
        system = B.assemble(kind, alpha, grid, tg, w.g_delta)
        y = B.solve_pint(system).trajectory
        ref = O.spectral_oracle(kind.value, alpha, 1, w.length, w.num_cells, w.horizon, w.num_steps, w.g_delta)
        assert rel(y, ref) <= O.parity_tolerance(tg.n_levels, system.omega)
        e_gpu = workloads.l2_error(y[0], w.z0, grid.h, 1)
        e_orc = workloads.l2_error(ref[0], w.z0, grid.h, 1)
        assert abs(e_gpu - e_orc) <= 5e-4 * abs(e_orc)


def test_deterministic_bits():
    w = workloads.make_small(2, 40, 24)
    grid = B.build_grid(2, w.length, w.num_cells)
    system = B.assemble(B.MethodKind.PINT_QBVM, 1e-3, grid, B.TimeGrid(w.horizon, w.num_steps), w.g_delta)
    a = B.solve_pint(system).trajectory
    b = B.solve_pint(system).trajectory
    assert np.array_equal(a, b)


# ----------------------------------------------------------------- residual

@pytest.mark.parametrize("dim,cells,steps", [(1, 16, 16), (2, 8, 8), (2, 20, 9), (3, 6, 5)])
@pytest.mark.parametrize("kind", [B.MethodKind.PINT_QBVM, B.MethodKind.PINT_MQBVM])
def test_device_residual_matches_host(dim, cells, steps, kind):
    w = workloads.make_small(dim, cells, steps, seed=17)
    grid = B.build_grid(dim, w.length, cells)
    system = B.assemble(kind, 1e-2, grid, B.TimeGrid(w.horizon, steps), w.g_delta)
    res = B.solve_pint(system)
    dev = res.residual_norm()
    host = B.residual(system, res.trajectory)[1]
    assert dev == pytest.approx(host, rel=1e-6, abs=1e-15)
    assert dev <= 1e-8 * max(1.0, abs(system.omega))
    # a perturbed trajectory gives the host residual too
    import torch
    y = res.trajectory_device.clone()
    y[1] += 1e-3
    from paper_2107_06381_b200.pint import device_residual_norm
    assert device_residual_norm(system, y) == pytest.approx(B.residual(system, y.cpu().numpy())[1], rel=1e-9)


# ----------------------------------------------------------------- device closed form / forward model (8(f) f2, f3)

@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("kind", list(B.MethodKind))
def test_device_spectral_oracle_vs_reference(golden, name, kind):
    dim, length, cells, horizon, steps, alpha = golden[f"case_{name}_params"]
    grid = B.build_grid(int(dim), length, int(cells))
    tg = B.TimeGrid(horizon, int(steps))
    data = golden[f"case_{name}_data"]
    y = B.solve_spectral_oracle(kind, alpha, grid, tg, data).trajectory
    ref = O.spectral_oracle(kind.value, alpha, int(dim), length, int(cells), horizon, int(steps), data)
    assert rel(y, ref) <= 1e-12
    if kind.is_circulant:
        assert rel(y, golden[f"oracle_{name}_{kind.value}"]) <= 1e-12


def test_device_march_forward_vs_reference(golden):
    """Per-mode forward model against the reference's N-step recursion."""
    g = B.march_forward(golden["march_z0"], B.TimeGrid(0.1, 8), B.build_grid(2, 1.0, 8))
    assert rel(g, golden["march_out"]) <= 1e-13
    g1 = B.march_forward(golden["c1_z0"], B.TimeGrid(1.0, 256), B.build_grid(1, np.pi, 256))
    assert rel(g1, golden["c1_g"]) <= 1e-13
    gt = B.march_forward(torch.from_numpy(golden["c1_z0"]).cuda(), B.TimeGrid(1.0, 256), B.build_grid(1, np.pi, 256))
    assert isinstance(gt, torch.Tensor) and gt.is_cuda


def _chunked_rel(a, b, rows=64):
    num = den = 0.0
    for i in range(0, a.shape[0], rows):
        num += torch.linalg.vector_norm(a[i:i + rows] - b[i:i + rows]).item() ** 2
        den += torch.linalg.vector_norm(b[i:i + rows]).item() ** 2
    return (num / den) ** 0.5


@pytest.mark.parametrize("name", ["c3", "c4"])
def test_full_size_solve_vs_device_oracle(name):
    """c3 / c4 at full size (1.07e9 / 4.26e9 DOF): the whole trajectory against
    the device closed form, and sampled levels against the host oracle."""
    from paper_2107_06381_b200 import pint as P
    w = workloads.make(name)
    grid = B.build_grid(w.dim, w.length, w.num_cells)
    tg = B.TimeGrid(w.horizon, w.num_steps)
    kind = B.MethodKind(w.kinds[0])
    system = B.assemble(kind, w.alphas[0], grid, tg, w.g_delta)
    y = B.solve_pint(system).trajectory_device
    P._plan_cache.clear()
    torch.cuda.empty_cache()
    # level 0, both sides of the first level-tile boundaries (8-level W tiles; the
    # level-group kernel's group and Z-slot boundaries at 8 and 16), the middle, and
    # the partial last level tile (n = 1025: levels 1024 = 128 * 8 alone; 257: 256)
    N = w.num_steps
    levels = np.array(sorted({0, 1, 7, 8, 15, 16, 17, N // 3, N - 9, N - 8, N - 1, N}))
    ref_host = O.spectral_oracle(kind.value, w.alphas[0], w.dim, w.length, w.num_cells, w.horizon, w.num_steps,
                                 w.g_delta, levels=levels)
    tol = O.parity_tolerance(tg.n_levels, system.omega)
    assert rel(y[torch.from_numpy(levels).cuda()].cpu().numpy(), ref_host) <= tol
    orc = B.solve_spectral_oracle(kind, w.alphas[0], grid, tg, w.g_delta).trajectory_device
    assert _chunked_rel(y, orc) <= tol
    del y, orc
    torch.cuda.empty_cache()


def test_c3_full_size_repeatable_bits():
    """c3 at full size, eight solves into fresh NaN-filled trajectories: every one
    bitwise equal to the first. The level-group kernel (k_dst_lvl4) orders its row
    and column tasks through device counters, mbarriers, L2 discards and
    setmaxnreg-split warpgroups; a race in any of them shows up as a differing
    (or NaN) element in one of 8.6e9."""
    from paper_2107_06381_b200 import pint as P
    w = workloads.make("c3")
    grid = B.build_grid(w.dim, w.length, w.num_cells)
    tg = B.TimeGrid(w.horizon, w.num_steps)
    system = B.assemble(B.MethodKind(w.kinds[0]), w.alphas[0], grid, tg, w.g_delta)
    plan = P.PintPlan(grid, tg.n_levels, tg.tau, system.omega)
    g = torch.from_numpy(w.g_delta).cuda()
    div = system.method.condition_divisor(tg.tau)
    first = plan.solve_device(g, div).clone()
    plan.check_status()
    assert bool(torch.isfinite(first[::64]).all())
    y = torch.empty_like(first)
    for _ in range(8):
        y.fill_(float("nan"))
        plan.solve_device(g, div, out=y)
        assert torch.equal(y, first)
    del y, first
    P._plan_cache.clear()
    torch.cuda.empty_cache()


@pytest.mark.parametrize("n", [9, 257, 513, 1025, 4097])
@pytest.mark.parametrize("dim", [1, 2, 3])
def test_fused_solve_reports_singular_column(n, dim):
    """A shift s_j = -mu_k makes (s_j - lap) singular (space.py:237-240): every
    pass-A kernel (generic, Rader 257, warp 513, Bluestein 1025; symmetric and
    plain tile lists) must report column j, also where j enters permuted."""
    import ctypes
    from paper_2107_06381_b200 import _lib, plans
    if dim == 3 and n > 513:
        pytest.skip("size")
    cells = 6
    grid = B.build_grid(dim, 1.0, cells)
    mu1 = B.space.mu1_of(grid)
    sp = plans.space_plan(dim, cells, mu1)
    diag = B.diagonalize(n, -0.3)
    shifts = diag.eigenvalues / 0.01
    k = [1, 2, 0][:dim]
    mu = mu1[k[0]] if dim == 1 else (mu1[k[0]] + mu1[k[1]] if dim == 2 else (mu1[k[0]] + mu1[k[1]]) + mu1[k[2]])
    j0 = 5
    shifts = shifts.copy()
    shifts[j0] = -mu
    tp = plans.time_plan(diag.gamma, shifts)
    lib = _lib.lib()
    g = torch.ones(grid.n_interior, dtype=torch.float64, device="cuda")
    y = torch.empty((n, grid.n_interior), dtype=torch.float64, device="cuda")
    nb = int(lib.bhcp_pint_workspace_bytes(sp.handle, tp.handle))
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    _lib.check(lib.bhcp_pint_solve(sp.handle, tp.handle, plans.ptr(g), 1.0, plans.ptr(y), plans.ptr(ws), nb,
                                   plans.stream_handle()), "bhcp_pint_solve")
    st = _lib.Status()
    status = ctypes.c_void_p(lib.bhcp_pint_status_ptr(sp.handle, tp.handle, plans.ptr(ws)))
    _lib.check(lib.bhcp_read_status(status, 1e-8, ctypes.byref(st), plans.stream_handle()), "bhcp_read_status")
    assert st.code == _lib.BHCP_ERR_SINGULAR_SHIFT
    assert st.bad_column == j0


@pytest.mark.parametrize("dim,cells,steps", [(1, 2, 1), (2, 2, 1), (3, 2, 2), (2, 3, 1), (1, 3, 2)])
def test_smallest_systems_vs_oracle(dim, cells, steps):
    """One interior point per axis and one or two time steps (n_levels = 2, 3)."""
    w = workloads.make_small(dim, cells, steps, seed=2)
    grid = B.build_grid(dim, w.length, cells)
    tg = B.TimeGrid(w.horizon, steps)
    for kind in (B.MethodKind.PINT_QBVM, B.MethodKind.PINT_MQBVM):
        system = B.assemble(kind, 1e-2, grid, tg, w.g_delta)
        y = B.solve_pint(system).trajectory
        ref = O.spectral_oracle(kind.value, 1e-2, dim, w.length, cells, w.horizon, steps, w.g_delta)
        assert y.shape == (steps + 1, (cells - 1) ** dim)
        assert rel(y, ref) <= O.parity_tolerance(tg.n_levels, system.omega)


@pytest.mark.parametrize("dim,cells,steps", [(2, 10, 256), (2, 8, 512), (2, 6, 1024), (3, 5, 256), (2, 512, 512)])
def test_zero_data_zero_trajectory_fast_kernels(dim, cells, steps):
    """test_pint.py::test_zero_data_gives_zero_solution on the specialised kernels:
    exact zeros and no residue error (0 <= tol * max(0, tiny))."""
    grid = B.build_grid(dim, 1.0, cells)
    system = B.assemble(B.MethodKind.PINT_MQBVM, 1e-2, grid, B.TimeGrid(0.5, steps), np.zeros(grid.n_interior))
    res = B.solve_pint(system)
    assert not res.trajectory_device.any().item()


@pytest.mark.parametrize("dim,cells,steps", [(1, 256, 256), (2, 40, 30), (2, 64, 512), (2, 40, 1024),
                                             (3, 12, 256), (2, 24, 4096), (3, 10, 1024)])
def test_graph_replay_matches_eager(dim, cells, steps):
    """PintPlan.capture on a FRESH plan (no eager solve before the capture: the
    symmetric tile lists of the Rader / Good-Thomas / prime-factor pass A are
    built at plan creation): the CUDA-graph replay of the fused solve gives the
    eager bits, and a new g copied into the captured input buffer is used."""
    w = workloads.make_small(dim, cells, steps, seed=9)
    grid = B.build_grid(dim, w.length, cells)
    tg = B.TimeGrid(w.horizon, steps)
    system = B.assemble(B.MethodKind.PINT_QBVM, 1e-3, grid, tg, w.g_delta)
    plan = B.PintPlan(grid, tg.n_levels, tg.tau, system.omega)
    div = system.method.condition_divisor(tg.tau)
    g = torch.from_numpy(w.g_delta).cuda()
    y = torch.empty((tg.n_levels, grid.n_interior), dtype=torch.float64, device="cuda")
    graph = plan.capture(g, div, y)
    eager = B.solve_pint(system).trajectory
    y.zero_()
    graph.replay()
    torch.cuda.synchronize()
    plan.check_status()
    assert np.array_equal(y.cpu().numpy(), eager)
    g.copy_(torch.from_numpy(2.0 * w.g_delta))
    graph.replay()
    torch.cuda.synchronize()
    assert np.array_equal(y.cpu().numpy(), 2.0 * eager)
