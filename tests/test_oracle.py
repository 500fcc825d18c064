"""Pin the CPU oracle (oracle/bhcp_oracle.py) against golden vectors produced
by the reference itself (tests/golden/make_golden.py) and against the
reference test-suite's known-answer cases. CPU only."""

import numpy as np
import pytest

from oracle import bhcp_oracle as O


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300)


@pytest.mark.parametrize("n", [1, 2, 4, 5, 9, 257, 513])
def test_diagonalize_bitwise(golden, n):
    gam, eig = O.diagonalize(n, complex(golden[f"diag_omega_{n}"]))
    assert np.array_equal(gam, golden[f"diag_gamma_{n}"])
    assert np.array_equal(eig, golden[f"diag_eig_{n}"])


def test_known_answer_eigenvalues_and_branch():
    # test_circulant.py:50-59
    _, eig = O.diagonalize(2, 2.0)
    assert np.allclose(np.sort(eig.real), [1 - np.sqrt(2), 1 + np.sqrt(2)], atol=1e-14)
    gam, _ = O.diagonalize(4, -1.0)
    assert np.allclose(gam, np.exp(1j * np.pi * np.arange(4) / 4), atol=1e-15)


@pytest.mark.parametrize("n", [2, 3, 4, 5, 8, 9, 17, 33, 65, 257, 513])
def test_time_transforms(golden, n):
    gam, _ = O.diagonalize(n, complex(golden[f"toeig_omega_{n}"]))
    s = O.to_eigenspace(golden[f"toeig_in_{n}"], gam)
    assert np.array_equal(s, golden[f"toeig_out_{n}"])
    back = O.from_eigenspace(s, gam)
    assert np.array_equal(back, golden[f"fromeig_out_{n}"])


@pytest.mark.parametrize("dim,cells", [(1, 2), (1, 8), (1, 16), (1, 33), (2, 3), (2, 7), (2, 8)])
def test_sine_transform_and_spectrum(golden, dim, cells):
    key = f"{dim}_{cells}"
    m = cells - 1
    assert np.array_equal(O.mode_eigenvalues(dim, np.pi, cells), golden[f"mu_{key}"])
    assert np.array_equal(O.sine_transform(golden[f"dst_real_in_{key}"], dim, m), golden[f"dst_real_out_{key}"])
    assert np.array_equal(O.sine_transform(golden[f"dst_cplx_in_{key}"], dim, m), golden[f"dst_cplx_out_{key}"])


@pytest.mark.parametrize("dim,cells", [(1, 8), (1, 16), (1, 33), (2, 7)])
def test_scipy_dst_pinned_by_dense_matrix(golden, dim, cells):
    m = cells - 1
    D = O.dst1_dense(m)
    x = golden[f"dst_real_in_{dim}_{cells}"]
    if dim == 1:
        dense = D @ x
    else:
        dense = (D @ x.reshape(m, m) @ D.T).ravel()
    assert rel(O.sine_transform(x, dim, m), dense) <= 1e-13


@pytest.mark.parametrize("dim,cells", [(1, 16), (2, 8)])
def test_shifted_solve(golden, dim, cells):
    rhs = golden[f"ssolve_rhs_{dim}_{cells}"]
    for i in range(3):
        s = complex(golden[f"ssolve_shift_{dim}_{cells}_{i}"])
        out = O.shifted_solve(s, rhs, dim, np.pi, cells)
        assert np.array_equal(out, golden[f"ssolve_out_{dim}_{cells}_{i}"])


def test_step_b(golden):
    out = O.step_b(golden["stepb_in"], golden["stepb_shifts"], 1, np.pi, 16)
    assert np.array_equal(out, golden["stepb_out"])


def test_step_b_reports_failing_column():
    mu1 = O.mu1(np.pi, 8)[0]
    with pytest.raises(O.SingularShift, match="column 2"):
        O.step_b(np.ones((7, 4), complex), np.array([1.0, 2.0, -mu1, 4.0]), 1, np.pi, 8)


CASES = ["1d_m8_n8", "1d_m16_n16", "1d_m4_n4", "2d_m6_n5", "2d_m8_n8"]


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("kind", ["pint-qbvm", "pint-mqbvm"])
def test_pint_and_oracle_match_reference(golden, name, kind):
    dim, length, cells, horizon, steps, alpha = golden[f"case_{name}_params"]
    dim, cells, steps = int(dim), int(cells), int(steps)
    data = golden[f"case_{name}_data"]
    traj, _ = O.solve_pint(kind, alpha, dim, length, cells, horizon, steps, data)
    assert np.array_equal(traj, golden[f"pint_{name}_{kind}"])
    orc = O.spectral_oracle(kind, alpha, dim, length, cells, horizon, steps, data)
    assert np.array_equal(orc, golden[f"oracle_{name}_{kind}"])


def test_c1_golden(golden):
    traj, ratio = O.solve_pint("pint-qbvm", 1e-3, 1, np.pi, 256, 1.0, 256, golden["c1_gdelta"])
    assert np.array_equal(traj, golden["c1_pint"])
    orc = O.spectral_oracle("pint-qbvm", 1e-3, 1, np.pi, 256, 1.0, 256, golden["c1_gdelta"])
    assert np.array_equal(orc, golden["c1_oracle"])
    assert rel(traj, orc) < 1e-12
    assert ratio < 1e-8


def test_march_forward_matches_reference(golden):
    out = O.march_forward(golden["march_z0"], 2, 1.0, 8, 0.1, 8)
    assert np.array_equal(out, golden["march_out"])
    spec = O.march_forward_spectral(golden["march_z0"], 2, 1.0, 8, 0.1, 8)
    assert rel(spec, golden["march_out"]) < 1e-13


def test_3d_restatement_reduces_to_1d_separable_modes():
    # a field that is a 1D mode along axes 2 and 3 times an arbitrary profile
    # along axis 1: the 3D closed form must factor into the 1D closed form with
    # mu shifted by the two fixed-axis eigenvalues. Pins the 3D spectrum sum
    # and axis order of the restatement (no reference counterpart).
    cells, m = 6, 5
    rng = np.random.default_rng(0)
    prof = rng.standard_normal(m)
    D = O.dst1_dense(m)
    e2, e3 = D[:, 1], D[:, 3]  # orthonormal sine modes k=2, k=4
    field = np.einsum("i,j,k->ijk", prof, e2, e3).ravel()
    coef = O.sine_transform(field, 3, m).reshape(m, m, m)
    # only k2=2, k3=4 survive, with the 1D transform of the profile on axis 1
    assert np.allclose(coef[:, 1, 3], D @ prof, atol=1e-13)
    coef[:, 1, 3] = 0
    assert np.abs(coef).max() < 1e-13
    mu = O.mode_eigenvalues(3, 1.0, cells).reshape(m, m, m)
    m1 = O.mu1(1.0, cells)
    assert np.array_equal(mu[:, 1, 3], (m1 + m1[1]) + m1[3])


def test_3d_pint_restatement_matches_closed_form():
    rng = np.random.default_rng(3)
    cells, steps = 5, 6
    data = rng.standard_normal((cells - 1) ** 3)
    for kind in ("pint-qbvm", "pint-mqbvm"):
        traj, _ = O.solve_pint(kind, 1e-2, 3, 1.0, cells, 0.05, steps, data)
        orc = O.spectral_oracle(kind, 1e-2, 3, 1.0, cells, 0.05, steps, data)
        assert rel(traj, orc) < 1e-12


@pytest.mark.parametrize("mesh", [(8, 8), (16, 8), (16, 16), (32, 32), (64, 64)])
@pytest.mark.parametrize("kind", [O.PINT_QBVM, O.PINT_MQBVM])
def test_residue_tripwire_like_reference(golden, mesh, kind):
    """circulant.py:182-189 on the reference's own noise-free ex1 rows (alpha =
    1e-12 fallback): the oracle raises exactly where the reference raised and
    reports the reference's residue ratio bit for bit."""
    M, N = mesh
    raised_ref, ratio_ref, alpha = golden[f"trip_ex1_{M}_{N}_{kind}"]
    data = golden[f"trip_ex1_{M}_{N}_data"]
    try:
        _, ratio = O.solve_pint(kind, alpha, 1, np.pi, M, 1.0, N, data)
        raised = False
    except O.ResidueError:
        raised = True
    tau = 1.0 / N
    gam, eig = O.diagonalize(N + 1, O.omega_of(kind, alpha, tau))
    s1 = O.to_eigenspace(O.rhs_block(data, kind, alpha, tau, N + 1).T, gam)
    s2 = O.step_b(s1, eig / tau, 1, np.pi, M)
    assert raised == bool(raised_ref)
    assert O.residue_ratio(s2, gam) == ratio_ref


def test_residue_no_raise_cases(golden):
    """BASELINE c1 does not trip the residue check (ratio 2e-13)."""
    traj, ratio = O.solve_pint(O.PINT_QBVM, 1e-3, 1, np.pi, 256, 1.0, 256, golden["c1_gdelta"])
    raised_ref, ratio_ref, _ = golden["trip_c1_pint-qbvm"]
    assert not raised_ref and ratio == ratio_ref


def test_reference_package_check_pins_port_timing_leg():
    """bench.py --impl reference runs the unmodified reference package (when it is
    installed under baseline/_ref) next to the oracle port on the same reduced
    problem: the trajectories must be bit-identical (pint.py:69-110)."""
    import importlib.util
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    if not (root / "baseline" / "_ref" / "bhcp").is_dir():
        pytest.skip("reference package not installed under baseline/_ref")
    spec = importlib.util.spec_from_file_location("bench_mod", root / "bench.py")
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    from paper_2107_06381_b200 import workloads

    w = workloads.make_small(2, 16, 40, kmax=4)
    out = bench.reference_package_check(w, "pint-mqbvm", 1e-2, 2, levels=9)
    assert out is not None and "unavailable" not in out, out
    assert out["levels"] == 9 and out["dof"] == 9 * 15 * 15
    assert out["port_vs_reference_rel_l2"] == 0.0
    assert out["workers_none"]["DOF_s"] > 0 and out["port_workers_all"]["DOF_s"] > 0
