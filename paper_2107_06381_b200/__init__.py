"""B200-native PinT QBVM/MQBVM direct solver (drop-in for the reference
``bhcp`` solve_pint path, arXiv:2107.06381).

Public names mirror the reference exports of pkg/src/bhcp/__init__.py:11-69
that belong to the hot path. Numerics run in libbhcp_b200.so (sm_100a); the
package has no CPU fallback.
"""

from .baseline import march_forward, solve_spectral_oracle
from .circulant import (
    CirculantDiagonalization,
    ImaginaryResidueError,
    TimeGrid,
    diagonalize,
    from_eigenspace,
    step_matrix,
    to_eigenspace,
)
from .methods import (
    AllAtOnceSystem,
    MethodKind,
    MethodSpec,
    SolveResult,
    alpha_rule,
    assemble,
    residual,
)
from .pint import PintPlan, solve_pint, solve_pint_unfused, step_b_parallel
from .space import (
    LaplacianOperator,
    SingularShiftError,
    SpatialGrid,
    SpatialSpectrum,
    build_grid,
    grid_norm,
    laplacian_eigenvalues,
    shifted_solve,
    sine_transform,
)

__version__ = "0.1.0"
