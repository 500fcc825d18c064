"""Error-path parity of the fused solve: the imaginary-residue tripwire of
from_eigenspace (circulant.py:182-189, tol 1e-8) on the device.

The reference raises ImaginaryResidueError on its own noise-free ex1 rows at
alpha = 1e-12 (bench.py:49-83 fallback; pkg/test_output.txt:118-119) and does
not raise on BASELINE c1 / c5. tests/golden/make_golden.py ran the reference
on every case below and recorded (raised, ||Im Y|| / ||Y||, alpha) as
``trip_<case>_<kind>``. The device must raise in exactly the reference's
cases, and its residue ratio -- ||Im|| / ||.|| of Gamma^-1 F* S2 as computed
on the device (the mode coefficients W carry the same Frobenius norms, Phi
being orthonormal) -- must lie within 10x of the reference's: both are
roundoff of the time transforms amplified by cond(Gamma).
"""

import numpy as np
import pytest
import torch

import paper_2107_06381_b200 as B
from paper_2107_06381_b200 import workloads

pytestmark = pytest.mark.gpu

KINDS = (B.MethodKind.PINT_QBVM, B.MethodKind.PINT_MQBVM)
EX1 = [(8, 8), (16, 8), (16, 16), (32, 32), (64, 64)]


def device_ratio(system):
    """(raised, device ratio) of solve_pint on `system`."""
    try:
        res = B.solve_pint(system)
        raised = False
    except B.ImaginaryResidueError:
        raised = True
    plan = B.pint.pint_plan(system.grid, system.timegrid, system.omega)
    st = plan.read_status(tol=1.0)   # the status block of that solve
    return raised, st.residue / st.norm, (None if raised else res.residue_ratio)


def check(golden, key, system):
    ref_raised, ref_ratio, _ = golden[key]
    raised, ratio, rr = device_ratio(system)
    msg = f"{key}: device ratio {ratio:.3e} (raised {raised}), reference {ref_ratio:.3e} (raised {bool(ref_raised)})"
    print(msg)
    assert raised == bool(ref_raised), msg
    assert ref_ratio / 10 <= ratio <= 10 * ref_ratio, msg
    if rr is not None:
        assert rr == pytest.approx(ratio, rel=1e-12)


@pytest.mark.parametrize("mesh", EX1)
@pytest.mark.parametrize("kind", KINDS)
def test_ex1_noise_free_rows_raise_like_reference(golden, mesh, kind):
    M, N = mesh
    data = golden[f"trip_ex1_{M}_{N}_data"]
    alpha = golden[f"trip_ex1_{M}_{N}_{kind.value}"][2]
    system = B.assemble(kind, alpha, B.build_grid(1, np.pi, M), B.TimeGrid(1.0, N), data)
    check(golden, f"trip_ex1_{M}_{N}_{kind.value}", system)


def test_c1_residue_like_reference(golden):
    system = B.assemble(B.MethodKind.PINT_QBVM, 1e-3, B.build_grid(1, np.pi, 256), B.TimeGrid(1.0, 256),
                        golden["c1_gdelta"])
    check(golden, "trip_c1_pint-qbvm", system)


@pytest.mark.parametrize("alpha", [1e-6, 1e-1])
@pytest.mark.parametrize("kind", KINDS)
def test_c5_residue_like_reference(golden, alpha, kind):
    w = workloads.make("c5")
    system = B.assemble(kind, alpha, B.build_grid(1, np.pi, 4096), B.TimeGrid(1.0, 4096), w.g_delta)
    check(golden, f"trip_c5_{alpha:g}_{kind.value}", system)


def test_unfused_dataflow_raises_like_reference(golden):
    """The literal 3-step device dataflow on the reference's tripwire rows."""
    for M, N in EX1:
        data = golden[f"trip_ex1_{M}_{N}_data"]
        for kind in KINDS:
            ref_raised = bool(golden[f"trip_ex1_{M}_{N}_{kind.value}"][0])
            system = B.assemble(kind, 1e-12, B.build_grid(1, np.pi, M), B.TimeGrid(1.0, N), data)
            try:
                B.solve_pint_unfused(system)
                raised = False
            except B.ImaginaryResidueError:
                raised = True
            assert raised == ref_raised, (M, N, kind.value)
    torch.cuda.synchronize()
