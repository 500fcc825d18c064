"""Driver integration: the reference's experiment driver with
its solve rebound to the device path.

CPU (this container, where /root/reference exists): the rebinding reaches
bench._solve, and without the CUDA library every row fails loudly instead of
falling back to the reference's numpy solve. GPU: the device solve and the
device oracle accept reference-shaped (duck-typed) systems and grids.
"""

import enum
import os
import sys
from dataclasses import dataclass

import numpy as np
import pytest

from oracle import bhcp_oracle as O

REF_SRC = "/root/reference/pkg/src"


@pytest.fixture
def bhcp():
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference package not present on this host")
    sys.path.insert(0, REF_SRC)
    try:
        import bhcp as mod
        yield mod
    finally:
        sys.path.remove(REF_SRC)


def test_install_rebinds_and_restores(bhcp):
    from paper_2107_06381_b200 import integration, pint as P
    import bhcp.bench as bench
    original = bench.solve_pint, bench.solve_spectral_oracle, bhcp.pint.solve_pint
    with integration.install(bhcp):
        assert bench.solve_pint is P.solve_pint and bhcp.pint.solve_pint is P.solve_pint
        assert bench.solve_spectral_oracle is not original[1]
    assert (bench.solve_pint, bench.solve_spectral_oracle, bhcp.pint.solve_pint) == original


def test_driver_rows_fail_loudly_without_gpu(bhcp, capsys):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2107_06381_b200 import integration
    from bhcp.bench import ExperimentConfig, run_experiment
    from bhcp.methods import MethodKind
    cfg = ExperimentConfig(example=1, methods=(MethodKind.PINT_QBVM,), solver="pint", meshes=((16, 16),),
                           eps_values=(1e-2,), seed=3)
    with integration.install(bhcp):
        reports = run_experiment(cfg)
    assert [r.status for r in reports] == ["error"]
    err = capsys.readouterr().err
    assert "libbhcp_b200" in err or "CUDA" in err


# ---------------------------------------------------------------- reference-shaped types on the GPU

class Kind(enum.Enum):
    PINT_QBVM = "pint-qbvm"
    PINT_MQBVM = "pint-mqbvm"

    @property
    def is_circulant(self):
        return True


@dataclass(frozen=True)
class Grid:
    dim: int
    length: float
    num_cells: int

    @property
    def h(self):
        return self.length / self.num_cells

    @property
    def n_interior(self):
        return (self.num_cells - 1) ** self.dim


@dataclass(frozen=True)
class Steps:
    horizon: float
    num_steps: int

    @property
    def tau(self):
        return self.horizon / self.num_steps

    @property
    def n_levels(self):
        return self.num_steps + 1


@dataclass(frozen=True)
class Spec:
    kind: Kind
    alpha: float


class System:
    def __init__(self, kind, alpha, grid, tg, data):
        self.method, self.grid, self.timegrid, self.data = Spec(kind, alpha), grid, tg, data
        div = tg.tau * alpha if kind is Kind.PINT_QBVM else alpha
        self.omega = -tg.tau / div
        self.n_levels, self.n_space = tg.n_levels, grid.n_interior


@pytest.mark.gpu
@pytest.mark.parametrize("kind", list(Kind))
def test_duck_typed_reference_system(kind):
    import paper_2107_06381_b200 as B
    grid, tg = Grid(2, 1.0, 24), Steps(0.1, 20)
    data = np.random.default_rng(5).standard_normal(grid.n_interior)
    res = B.solve_pint(System(kind, 1e-3, grid, tg, data))
    ref = O.spectral_oracle(kind.value, 1e-3, 2, 1.0, 24, 0.1, 20, data)
    tol = O.parity_tolerance(tg.n_levels, -tg.tau / (tg.tau * 1e-3 if kind is Kind.PINT_QBVM else 1e-3))
    assert np.linalg.norm(res.trajectory - ref) / np.linalg.norm(ref) <= tol
    assert res.status == "ok" and res.solver == "pint"
    assert set(res.timings) == {"step_a", "step_b", "step_c", "total"}
    assert res.residual_norm() <= 1e-9
    orc = B.solve_spectral_oracle(kind, 1e-3, grid, tg, data)
    assert np.linalg.norm(orc.initial_state - ref[0]) / np.linalg.norm(ref[0]) <= 1e-12


# ------------------------------------------------- the reference driver itself on the B200 (f4)

def _reference_package():
    """The reference package as test data: the read-only source tree where it
    exists (this container), else the copy pip-installed into baseline/_ref
    (git-ignored; it travels to the GPU box with the snapshot). Never imported by
    the product package."""
    from pathlib import Path

    for root in (REF_SRC, str(Path(__file__).resolve().parents[1] / "baseline" / "_ref")):
        if os.path.isdir(os.path.join(root, "bhcp")):
            return root
    return None


@pytest.mark.gpu
@pytest.mark.parametrize("example,meshes", [(1, ((32, 32), (64, 64))), (2, ((16, 16),))])
def test_reference_driver_rows_on_device(example, meshes, tmp_path):
    """bhcp.bench.run_experiment (bench.py:172-272) with its solve rebound to the
    device by integration.install, against the same experiment on the reference's
    own numpy path: every row ok, CSV error_l2 equal to 3 significant digits (the
    north-star bar for the reconstruction error), residual of the device row at
    the reference's level. The reference's own fixed-alpha tripwire row (M, N) =
    (16, 8) at alpha 1e-12 must fail on both paths (ImaginaryResidueError,
    circulant.py:182-189)."""
    root = _reference_package()
    if root is None:
        pytest.skip("reference package not available (neither /root/reference nor baseline/_ref)")
    sys.path.insert(0, root)
    try:
        import bhcp
        from bhcp.bench import ExperimentConfig, emit_csv, parse_csv, run_experiment
        from bhcp.methods import MethodKind

        from paper_2107_06381_b200 import integration

        kinds = (MethodKind.PINT_QBVM, MethodKind.PINT_MQBVM)
        cfg = ExperimentConfig(example=example, methods=kinds, solver="pint", meshes=meshes, eps_values=(1e-2, 1e-3),
                               seed=11)
        cpu = run_experiment(cfg)
        with integration.install(bhcp):
            dev = run_experiment(cfg)
        emit_csv(dev, str(tmp_path / "dev.csv"))
        emit_csv(cpu, str(tmp_path / "cpu.csv"))
        rd, rc = parse_csv(str(tmp_path / "dev.csv")), parse_csv(str(tmp_path / "cpu.csv"))
        assert len(rd) == len(rc) == len(kinds) * len(meshes) * 2
        for a, b in zip(rd, rc):
            assert a.status == b.status == "ok", (a.status, b.status)
            assert float(f"{a.error_l2:.3g}") == float(f"{b.error_l2:.3g}"), (a.error_l2, b.error_l2)
            assert a.residual <= max(10 * b.residual, 1e-9)
        trip = ExperimentConfig(example=1, methods=kinds, solver="pint", meshes=((16, 8),), eps_values=(1e-2,),
                                seed=3, alpha_rule="fixed:1e-12")
        with integration.install(bhcp):
            dev_trip = run_experiment(trip)
        assert [r.status for r in run_experiment(trip)] == [r.status for r in dev_trip]
    finally:
        sys.path.remove(root)
        for k in [k for k in sys.modules if k == "bhcp" or k.startswith("bhcp.")]:
            del sys.modules[k]
