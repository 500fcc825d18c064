"""Route the reference experiment driver to the device solver.

The reference driver picks the solver in ``bench._solve`` (bench.py:196-209),
calling the names ``solve_pint`` and ``solve_spectral_oracle`` bound in the
``bhcp.bench`` module. ``install`` rebinds them (and ``bhcp.pint.solve_pint``,
``bhcp.solve_pint``) to the device implementations, so ``bhcp run --solver
pint`` keeps its CSV schema, seeds, alpha rules, ``l2_error`` scoring and
profile files (bench.py:154-162, 212-334) and only the solve moves to the
GPU. The device functions accept the reference's own ``AllAtOnceSystem``,
``SpatialGrid``, ``TimeGrid`` and ``MethodKind`` (duck-typed) and return a
``SolveResult`` with the attributes the driver reads: ``status``,
``initial_state``, ``timings`` (step_a/b/c/total) and ``residual_norm()``
(device stencil pass, f1).

There is no fallback: on a host without the CUDA library the rebound solve
raises ``NativeLibraryError`` and the driver records the row as an error.

    import bhcp
    from paper_2107_06381_b200 import integration
    with integration.install(bhcp):
        reports = bhcp.bench.run_experiment(config)
"""

from __future__ import annotations

import importlib

from .baseline import solve_spectral_oracle as _device_oracle
from .pint import solve_pint as _device_solve_pint


class Installation:
    """Handle returned by ``install``; ``uninstall()`` (or leaving the ``with``
    block) restores the reference bindings."""

    def __init__(self, patches):
        self._patches = patches  # [(module, name, original)]

    def uninstall(self) -> None:
        for module, name, original in reversed(self._patches):
            setattr(module, name, original)
        self._patches = []

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.uninstall()
        return False


def install(bhcp, oracle: bool = True) -> Installation:
    """Rebind the reference package's PinT solve (and, with ``oracle``, its
    closed-form solver) to the device implementations."""
    bench = importlib.import_module(bhcp.__name__ + ".bench")
    pint = importlib.import_module(bhcp.__name__ + ".pint")
    targets = [(bench, "solve_pint", _device_solve_pint), (pint, "solve_pint", _device_solve_pint)]
    if hasattr(bhcp, "solve_pint"):
        targets.append((bhcp, "solve_pint", _device_solve_pint))
    if oracle:
        targets.append((bench, "solve_spectral_oracle", _device_oracle))
    patches = []
    for module, name, fn in targets:
        patches.append((module, name, getattr(module, name)))
        setattr(module, name, fn)
    return Installation(patches)
