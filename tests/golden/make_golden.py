"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container only (the reference checkout is not on the GPU
box):  python tests/golden/make_golden.py
It imports ``bhcp`` read-only from /root/reference/pkg/src and writes
``tests/golden/golden.npz``. Every array in that file is an output of the
reference's own code path on seeded inputs (names say which function):

  diag_*        circulant.diagonalize            (circulant.py:134-153)
  toeig_*       circulant.to_eigenspace          (circulant.py:156-164)
  fromeig_*     circulant.from_eigenspace        (circulant.py:167-190)
  dst_*         space.sine_transform             (space.py:223-231)
  mu_*          space.laplacian_eigenvalues      (space.py:202-220)
  ssolve_*      space.shifted_solve              (space.py:249-283)
  stepb_*       pint.step_b_parallel             (pint.py:26-66)
  pint_*        pint.solve_pint                  (pint.py:69-110)
  oracle_*      baseline.solve_spectral_oracle   (baseline.py:67-112)
  march_*       baseline.march_forward           (baseline.py:115-129)
  c1_*          BASELINE config 1 inputs/outputs (seeded, see workloads.py)
  trip_*        the imaginary-residue tripwire of from_eigenspace (circulant.py:
                182-189): the reference's raise / no-raise decision and its
                residue ratio ||Im Y|| / ||Y|| for the noise-free ex1 rows that
                the reference driver records as failed (pkg/test_output.txt:
                118-119; alpha = the 1e-12 fallback of bench.py:49-83), and for
                BASELINE c1 and c5 pint-qbvm at alpha = 1e-6 (no raise)
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from bhcp.baseline import march_forward, solve_spectral_oracle  # noqa: E402
from bhcp.circulant import TimeGrid, diagonalize, from_eigenspace, to_eigenspace  # noqa: E402
from bhcp.methods import MethodKind, assemble  # noqa: E402
from bhcp.pint import solve_pint, step_b_parallel  # noqa: E402
from bhcp.space import build_grid, laplacian_eigenvalues, shifted_solve, sine_transform  # noqa: E402
from bhcp.analysis import get_problem  # noqa: E402
from bhcp.bench import resolve_alpha  # noqa: E402
from bhcp.circulant import ImaginaryResidueError  # noqa: E402

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2107_06381_b200 import workloads  # noqa: E402  (host-side seeded input generator)

OUT = Path(__file__).with_name("golden.npz")
g = {}

# --- diagonalize
for n, om in [(1, 3.0), (2, 2.0), (4, -1.0), (5, -1e-4), (9, -10.0), (257, -1000.0), (513, -0.01953125)]:
    d = diagonalize(n, om)
    g[f"diag_gamma_{n}"] = d.gamma
    g[f"diag_eig_{n}"] = d.eigenvalues
    g[f"diag_omega_{n}"] = np.array(om)

# --- time transforms (general blocks, time on the trailing axis)
rng = np.random.default_rng(101)
for n, om in [(2, -1e4), (3, -1.0), (4, -0.7), (5, 2.0), (8, -1e-4), (9, -10.0), (17, -3.0),
              (33, -1e3), (65, -0.5), (257, -1e3), (513, -0.01953125)]:
    d = diagonalize(n, om)
    blk = rng.standard_normal((6, n))
    s = to_eigenspace(blk, d)
    g[f"toeig_in_{n}"] = blk
    g[f"toeig_omega_{n}"] = np.array(om)
    g[f"toeig_out_{n}"] = s
    g[f"fromeig_out_{n}"] = from_eigenspace(s, d)

# --- sine transforms and spectra
for dim, cells in [(1, 2), (1, 8), (1, 16), (1, 33), (2, 3), (2, 7), (2, 8)]:
    grid = build_grid(dim, np.pi, cells)
    x = rng.standard_normal(grid.n_interior)
    z = rng.standard_normal(grid.n_interior) + 1j * rng.standard_normal(grid.n_interior)
    key = f"{dim}_{cells}"
    g[f"dst_real_in_{key}"] = x
    g[f"dst_real_out_{key}"] = sine_transform(grid, x)
    g[f"dst_cplx_in_{key}"] = z
    g[f"dst_cplx_out_{key}"] = sine_transform(grid, z)
    g[f"mu_{key}"] = laplacian_eigenvalues(grid).mode_eigenvalues

# --- shifted solves
for dim, cells in [(1, 16), (2, 8)]:
    grid = build_grid(dim, np.pi, cells)
    rhs = rng.standard_normal(grid.n_interior) + 1j * rng.standard_normal(grid.n_interior)
    for i, s in enumerate([4.0, 3.0 + 2.0j, -0.5 + 40.0j]):
        g[f"ssolve_rhs_{dim}_{cells}"] = rhs
        g[f"ssolve_shift_{dim}_{cells}_{i}"] = np.array(s)
        g[f"ssolve_out_{dim}_{cells}_{i}"] = shifted_solve(grid, s, rhs)

# --- step b (test_pint.py:104-112 case)
grid = build_grid(1, np.pi, 16)
d = diagonalize(9, -10.0)
blk = rng.standard_normal((15, 9)) + 1j * rng.standard_normal((15, 9))
g["stepb_in"] = blk
g["stepb_shifts"] = d.eigenvalues / 0.125
g["stepb_out"] = step_b_parallel(grid, blk, d.eigenvalues / 0.125)

# --- full solves, small 1D/2D, both kinds
cases = [
    ("1d_m8_n8", 1, np.pi, 8, 1.0, 8, 0.1),
    ("1d_m16_n16", 1, np.pi, 16, 1.0, 16, 1e-3),
    ("1d_m4_n4", 1, np.pi, 4, 1.0, 4, 1e-6),
    ("2d_m6_n5", 2, np.pi, 6, 1.0, 5, 1e-2),
    ("2d_m8_n8", 2, 1.0, 8, 0.1, 8, 1e-3),
]
for name, dim, length, cells, horizon, steps, alpha in cases:
    grid = build_grid(dim, length, cells)
    tg = TimeGrid(horizon, steps)
    data = np.random.default_rng(4).standard_normal(grid.n_interior)
    g[f"case_{name}_data"] = data
    g[f"case_{name}_params"] = np.array([dim, length, cells, horizon, steps, alpha])
    for kind in (MethodKind.PINT_QBVM, MethodKind.PINT_MQBVM):
        sysm = assemble(kind, alpha, grid, tg, data)
        g[f"pint_{name}_{kind.value}"] = solve_pint(sysm).trajectory
        g[f"oracle_{name}_{kind.value}"] = solve_spectral_oracle(kind, alpha, grid, tg, data).trajectory

# --- march_forward (data generator) on a small 2D grid
grid = build_grid(2, 1.0, 8)
z0 = rng.standard_normal(grid.n_interior)
g["march_z0"] = z0
g["march_out"] = march_forward(z0, TimeGrid(0.1, 8), grid)

# --- BASELINE config 1, generated with the reference's own march_forward
#     (seed convention: rng = default_rng(seed); coefficients first, then eps)
seed, delta, alpha = 1, 1e-3, 1e-3
grid = build_grid(1, np.pi, 256)
tg = TimeGrid(1.0, 256)
rng1 = np.random.default_rng(seed)
k = np.arange(1, 9)
coef = rng1.standard_normal(8) / k**2
x = grid.interior_coords()[0]
z0 = np.sin(np.outer(x, k)) @ coef
gclean = march_forward(z0, tg, grid)
eps = rng1.standard_normal(grid.n_interior)
gdelta = gclean + delta * eps / np.linalg.norm(eps) * np.linalg.norm(gclean)
sysm = assemble(MethodKind.PINT_QBVM, alpha, grid, tg, gdelta)
res = solve_pint(sysm)
g["c1_z0"] = z0
g["c1_g"] = gclean
g["c1_gdelta"] = gdelta
g["c1_pint"] = res.trajectory
g["c1_oracle"] = solve_spectral_oracle(MethodKind.PINT_QBVM, alpha, grid, tg, gdelta).trajectory



# --- the imaginary-residue tripwire (circulant.py:182-189)
def residue_case(key, kind, alpha, grid, tg, data):
    """Run the reference solve_pint; record whether it raised and its ratio."""
    sysm = assemble(kind, alpha, grid, tg, data)
    try:
        solve_pint(sysm)
        raised = 0
    except ImaginaryResidueError:
        raised = 1
    # the same quantity the reference tests: ||Im Y|| / ||Y|| of Y = apply_basis(S2)
    diag = diagonalize(tg.n_levels, sysm.omega)
    s1 = to_eigenspace(sysm.rhs().reshape(tg.n_levels, grid.n_interior).T, diag)
    s2 = step_b_parallel(grid, s1, diag.eigenvalues / tg.tau)
    out = diag.apply_basis(s2)
    ratio = np.linalg.norm(out.imag) / max(np.linalg.norm(out), np.finfo(float).tiny)
    g[f"trip_{key}_{kind.value}"] = np.array([raised, ratio, alpha])


ex1 = get_problem("ex1")
trip_meshes = [(8, 8), (16, 8), (16, 16), (32, 32), (64, 64)]
for M, N in trip_meshes:
    grid = build_grid(1, np.pi, M)
    tg = TimeGrid(1.0, N)
    data = ex1.final_on_grid(grid)
    g[f"trip_ex1_{M}_{N}_data"] = data
    for kind in (MethodKind.PINT_QBVM, MethodKind.PINT_MQBVM):
        residue_case(f"ex1_{M}_{N}", kind, resolve_alpha("auto", kind, 0.0, tg.tau), grid, tg, data)
residue_case("c1", MethodKind.PINT_QBVM, 1e-3, build_grid(1, np.pi, 256), TimeGrid(1.0, 256), gdelta)
w5 = workloads.make("c5")
for alpha in (1e-6, 1e-1):
    for kind in (MethodKind.PINT_QBVM, MethodKind.PINT_MQBVM):
        residue_case(f"c5_{alpha:g}", kind, alpha, build_grid(1, np.pi, 4096), TimeGrid(1.0, 4096), w5.g_delta)

np.savez_compressed(OUT, **g)
print(f"wrote {OUT} with {len(g)} arrays, {OUT.stat().st_size / 1e6:.2f} MB")
