"""Host-side logic of the device package: plans inputs, grids, methods, error
semantics that trigger before any device work, and the seeded workloads.
CPU only."""

import numpy as np
import pytest

import paper_2107_06381_b200 as B
from paper_2107_06381_b200 import workloads


def test_diagonalize_is_bitwise_reference(golden):
    for n in (1, 2, 4, 5, 9, 257, 513):
        d = B.diagonalize(n, complex(golden[f"diag_omega_{n}"]))
        assert np.array_equal(d.gamma, golden[f"diag_gamma_{n}"])
        assert np.array_equal(d.eigenvalues, golden[f"diag_eig_{n}"])


@pytest.mark.parametrize("dim,cells", [(1, 2), (1, 8), (1, 33), (2, 3), (2, 8)])
def test_spectrum_is_bitwise_reference(golden, dim, cells):
    spec = B.laplacian_eigenvalues(B.build_grid(dim, np.pi, cells))
    assert np.array_equal(spec.mode_eigenvalues, golden[f"mu_{dim}_{cells}"])


def test_grid_and_timegrid_validation():
    with pytest.raises(ValueError):
        B.build_grid(4, 1.0, 4)
    with pytest.raises(ValueError):
        B.build_grid(1, 0.0, 4)
    with pytest.raises(ValueError):
        B.build_grid(1, 1.0, 1)
    assert B.build_grid(3, 1.0, 256).n_interior == 255**3
    with pytest.raises(ValueError):
        B.TimeGrid(0.0, 4)
    with pytest.raises(ValueError):
        B.TimeGrid(1.0, 0)
    assert B.TimeGrid(1.0, 8).n_levels == 9


def test_method_scalars():
    tau = 0.125
    q = B.MethodSpec(B.MethodKind.PINT_QBVM, 0.1)
    mq = B.MethodSpec(B.MethodKind.PINT_MQBVM, 0.1)
    assert q.condition_divisor(tau) == tau * 0.1
    assert mq.condition_divisor(tau) == 0.1
    assert q.omega(tau) == -tau / (tau * 0.1)
    assert mq.omega(tau) == -tau / 0.1
    assert B.MethodSpec(B.MethodKind.QBVM, 0.1).omega(tau) is None
    with pytest.raises(ValueError):
        B.MethodSpec(B.MethodKind.PINT_QBVM, 0.0)


@pytest.mark.parametrize("kind", [B.MethodKind.QBVM, B.MethodKind.MQBVM])
def test_classic_kinds_rejected_before_device(kind):
    grid = B.build_grid(1, np.pi, 8)
    system = B.assemble(kind, 0.1, grid, B.TimeGrid(1.0, 8), np.ones(7))
    with pytest.raises(ValueError):
        B.solve_pint(system)


def test_rhs_layout_and_apply_identity():
    grid = B.build_grid(2, 1.0, 5)
    tg = B.TimeGrid(0.1, 4)
    data = np.arange(16.0)
    system = B.assemble(B.MethodKind.PINT_QBVM, 0.01, grid, tg, data)
    rhs = system.rhs().reshape(tg.n_levels, -1)
    assert np.array_equal(rhs[0], data / (tg.tau * 0.01))
    assert not rhs[1:].any()
    # the spectral oracle solution satisfies the assembled system
    from oracle import bhcp_oracle as O
    y = O.spectral_oracle("pint-qbvm", 0.01, 2, 1.0, 5, 0.1, 4, data)
    _, rel = B.residual(system, y)
    assert rel < 1e-12


def test_workload_c1_matches_reference_march_forward(golden):
    w = workloads.make("c1")
    assert np.array_equal(w.z0, golden["c1_z0"])
    assert np.linalg.norm(w.g - golden["c1_g"]) <= 1e-13 * np.linalg.norm(golden["c1_g"])
    assert np.linalg.norm(w.g_delta - golden["c1_gdelta"]) <= 1e-13 * np.linalg.norm(golden["c1_gdelta"])


def test_workload_noise_is_relative_delta():
    w = workloads.make("c1")
    assert abs(np.linalg.norm(w.g_delta - w.g) / np.linalg.norm(w.g) - w.delta) < 1e-12


def test_workload_2d_construction_small():
    w = workloads.make_small(2, 8, 8)
    assert w.z0.shape == (49,)
    from oracle import bhcp_oracle as O
    g_ref = O.march_forward(w.z0, 2, w.length, w.num_cells, w.horizon, w.num_steps)
    assert np.linalg.norm(w.g - g_ref) <= 1e-13 * np.linalg.norm(g_ref)
