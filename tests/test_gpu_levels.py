"""Device parity of the spatial level passes of the fused solve (B200 only).

The fused solve ends with y[t, :] = Phi W[t, :] (pint.py:94-99 with the
inverse DST moved after the time transform). For m + 1 in
{256, 512} the strided axes run in place on the blocked W (k_dst_wax /
k_dst_wax2, TMA tiles) and the last axis moves W -> y (k_dst_blk3); for 1024
the last axis moves W -> y first (k_dst_blk4, two warps per line pair) and the
strided axis runs on y (k_dst_cols3); in 2D the solve runs both as one
persistent level-group kernel over L2-resident level tiles (k_dst_lvl4,
bhcp_pint_levels_fused). These
tests feed seeded random blocked W -- with NaN in the padding levels of the
last level tile, which pass A never writes -- through every entry point that
runs those kernels and compare with the oracle's orthonormal DST
(oracle.fused_pass_b, scipy.fft.dst type 1) at 1e-13 relative L2.
"""

import numpy as np
import pytest
import torch

import paper_2107_06381_b200 as B
from oracle import bhcp_oracle as O
from paper_2107_06381_b200 import _lib, plans
from paper_2107_06381_b200.space import plan_for

pytestmark = pytest.mark.gpu

TB = 8   # levels per W block (fastk::kTBL)


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def blocked(F, dim, m):
    """Level-major F (L, m^dim) -> blocked W (k1, level tile, rest, 8 levels), NaN padding."""
    L = F.shape[0]
    nt = (L + TB - 1) // TB
    P1 = m ** (dim - 1)
    W = np.full((m, nt, P1, TB), np.nan)
    Fr = F.reshape(L, m, P1)
    for t in range(L):
        W[:, t // TB, :, t % TB] = Fr[t]
    return W.reshape(-1)


def run_levels(sp, W_host, L, dim, m, how):
    lib = _lib.lib()
    sh = plans.stream_handle()
    W = torch.from_numpy(W_host).cuda()
    y = torch.full((L, m ** dim), np.nan, dtype=torch.float64, device="cuda")
    if how == "levels":
        _lib.check(lib.bhcp_pint_levels(sp, plans.ptr(W), plans.ptr(y), L, sh), "levels")
    elif how == "passes":
        # the bench's phase-by-phase order: strided axes on W, then the last axis
        # (m + 1 = 1024: the last axis W -> y, then the strided axes on y)
        if lib.bhcp_pint_w_passes_supported(sp):
            for a in range(dim - 1):
                _lib.check(lib.bhcp_pint_w_pass(sp, plans.ptr(W), L, a, sh), "w pass")
            _lib.check(lib.bhcp_pint_level_pass(sp, plans.ptr(W), None, plans.ptr(y), L, 0, sh), "level pass 0")
        else:
            for p in range(dim):
                _lib.check(lib.bhcp_pint_level_pass(sp, plans.ptr(W), None, plans.ptr(y), L, p, sh), "level pass")
    elif how == "fused":
        # the one-kernel level-group pass (k_dst_lvl4 where the sync size is > 0)
        nb = lib.bhcp_pint_levels_sync_bytes(sp, L)
        sync = torch.full((max(nb, 8) // 4 + 1,), 12345, dtype=torch.int32, device="cuda")   # the call zeroes it
        _lib.check(lib.bhcp_pint_levels_fused(sp, plans.ptr(W), plans.ptr(y), L, plans.ptr(sync), sh), "levels_fused")
    elif how == "blocked":
        # an all-to-all receive buffer at the uniform k1 stride (koff NULL): the TMA passes
        _lib.check(lib.bhcp_pint_levels_blocked(sp, plans.ptr(W), None, plans.ptr(y), L, sh), "levels_blocked")
    else:
        # an explicit, non-uniform k1 -> block table: the k1 blocks stored in reverse
        # order; the general passes honour it
        nt = (L + TB - 1) // TB
        blk = nt * m ** (dim - 1) * TB
        Wr = W.view(m, blk).flip(0).contiguous().view(-1)
        koff = (m - 1 - torch.arange(m, dtype=torch.int64, device="cuda")) * blk
        _lib.check(lib.bhcp_pint_levels_blocked(sp, plans.ptr(Wr), plans.ptr(koff), plans.ptr(y), L, sh),
                   "levels_blocked table")
    torch.cuda.synchronize()
    return y.cpu().numpy()


@pytest.mark.parametrize("dim,cells,L", [(2, 512, 1), (2, 512, 7), (2, 512, 8), (2, 512, 9), (2, 512, 13),
                                         (2, 512, 16), (2, 256, 5), (2, 256, 8), (2, 256, 11), (3, 256, 1),
                                         (3, 256, 3), (2, 1024, 1), (2, 1024, 6), (2, 1024, 9), (2, 1024, 16),
                                         (2, 1024, 23), (2, 1024, 41)])
def test_level_passes_vs_oracle(dim, cells, L):
    grid = B.build_grid(dim, 1.0, cells)
    m = cells - 1
    plan = plan_for(grid)
    lib = _lib.lib()
    wside = lib.bhcp_pint_w_passes_supported(plan.handle) == 1
    assert wside == (cells in (256, 512))
    rng = np.random.default_rng(1000 * dim + 10 * cells + L)
    F = rng.standard_normal((L, m ** dim))
    ref = O.fused_pass_b(F, dim, m)
    W = blocked(F, dim, m)
    y = run_levels(plan.handle, W, L, dim, m, "levels")
    assert np.isfinite(y).all(), "padding NaN leaked into a valid level"
    err = rel(y, ref)
    assert err <= 1e-13, f"rel-L2 {err:.2e}"
    # the same kernels driven pass by pass (bench order) and through the
    # all-to-all receive-buffer entry point give the same bits
    assert np.array_equal(run_levels(plan.handle, W, L, dim, m, "passes"), y)
    assert np.array_equal(run_levels(plan.handle, W, L, dim, m, "blocked"), y)
    yt = run_levels(plan.handle, W, L, dim, m, "table")
    assert rel(yt, ref) <= 1e-13, "explicit block table"
    # the level-group kernel (m + 1 = 1024 in 2D; elsewhere the same passes as above)
    fused = lib.bhcp_pint_levels_sync_bytes(plan.handle, L) > 0
    assert fused == (dim == 2 and cells == 1024)
    yf = run_levels(plan.handle, W, L, dim, m, "fused")
    assert np.isfinite(yf).all(), "padding NaN leaked into a valid level (fused)"
    assert rel(yf, ref) <= 1e-13, f"fused rel-L2 {rel(yf, ref):.2e}"
    if not fused:
        assert np.array_equal(yf, y)
    else:
        # deterministic: a second run gives the same bits
        assert np.array_equal(run_levels(plan.handle, W, L, dim, m, "fused"), yf)


@pytest.mark.parametrize("dim,cells", [(2, 512), (3, 256)])
def test_w_pass_single_axis_vs_oracle(dim, cells):
    """bhcp_pint_w_pass alone: the DST along spatial axis a of every level, in place on W."""
    import scipy.fft as sf

    grid = B.build_grid(dim, 1.0, cells)
    m = cells - 1
    plan = plan_for(grid)
    lib = _lib.lib()
    L = 10 if dim == 2 else 2
    rng = np.random.default_rng(7 + dim)
    F = rng.standard_normal((L, m ** dim))
    for a in range(dim - 1):
        W = torch.from_numpy(blocked(F, dim, m)).cuda()
        _lib.check(lib.bhcp_pint_w_pass(plan.handle, plans.ptr(W), L, a, plans.stream_handle()), "w pass")
        torch.cuda.synchronize()
        nt = (L + TB - 1) // TB
        Wd = W.cpu().numpy().reshape(m, nt, m ** (dim - 1), TB)
        got = np.stack([Wd[:, t // TB, :, t % TB].reshape(-1) for t in range(L)])
        ref = sf.dst(F.reshape((L,) + (m,) * dim), type=1, norm="ortho", axis=1 + a).reshape(L, -1)
        assert rel(got, ref) <= 1e-13


def test_w_pass_rejects_unsupported():
    lib = _lib.lib()
    plan = plan_for(B.build_grid(2, 1.0, 1024))   # c3 keeps the y-side strided pass
    assert lib.bhcp_pint_w_passes_supported(plan.handle) == 0
    W = torch.zeros(8 * 1023 * 1023, dtype=torch.float64, device="cuda")
    assert lib.bhcp_pint_w_pass(plan.handle, plans.ptr(W), 1, 0, plans.stream_handle()) == _lib.BHCP_ERR_INVALID
    plan2 = plan_for(B.build_grid(2, 1.0, 512))
    assert lib.bhcp_pint_w_pass(plan2.handle, plans.ptr(W), 1, 1, plans.stream_handle()) == _lib.BHCP_ERR_INVALID
