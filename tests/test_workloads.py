"""The seeded BASELINE inputs (paper_2107_06381_b200/workloads.py) against the
reference's own data generator: g = march_forward(z0) (baseline.py:115-129),
recorded for config 1 in tests/golden/golden.npz by make_golden.py. CPU only."""

import numpy as np

from paper_2107_06381_b200 import workloads


def test_c1_inputs_match_reference_march_forward(golden):
    w = workloads.make("c1")
    # same seed convention (coefficients first, then eps): z0 bit-identical
    assert np.array_equal(w.z0, golden["c1_z0"])
    # per-mode forward model == the reference's N sequential shifted solves to roundoff
    g_ref = golden["c1_g"]
    assert np.linalg.norm(w.g - g_ref) / np.linalg.norm(g_ref) <= 1e-12
    assert np.linalg.norm(w.g_delta - golden["c1_gdelta"]) / np.linalg.norm(golden["c1_gdelta"]) <= 1e-12


def test_noise_is_exactly_relative_delta():
    for name in ("c1", "c2"):
        w = workloads.make(name)
        assert abs(np.linalg.norm(w.g_delta - w.g) / np.linalg.norm(w.g) - w.delta) <= 1e-12 * w.delta


def test_config_shapes():
    for name, dof in (("c1", 255 * 257), ("c2", 511**2 * 513), ("c3", 1023**2 * 1025), ("c4", 255**3 * 257),
                      ("c5", 4095 * 4097)):
        dim, length, M, T, N, kinds, alphas, delta, kmax = workloads.CONFIGS[name]
        assert (M - 1) ** dim * (N + 1) == dof
    assert len(workloads.CONFIGS["c5"][6]) == 64
