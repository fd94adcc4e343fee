"""B200-native solve phase of the two-level Schwarz / H_k-GenEO preconditioned
weighted GMRES for indefinite Helmholtz (arXiv 2406.06283).

Drop-in for the reference package ``helmdd``'s solve path:

    precond = factorize(forms, dec, coarse)            # schwarz.py:74
    x, rep = weighted_gmres(precond.as_operator("T"),  # cli.py:297-307
                            precond.apply(f), weight=forms.dk, rtol=1e-6)

The setup modules (fem, decomp, coarse, factor, problems) restate the
reference's setup on the host; the solve runs in libhelmgpu.so
(csrc/, include/helmgpu.h) on sm_100a.
"""

from .coarse import (
    CoarseSpace,
    LocalGevp,
    LocalGevpResult,
    ModeSelection,
    assemble_local_gevp,
    build_coarse_space,
    select_modes,
    solve_gevp_lanczos,
    solve_indefinite_gevp,
    spectrum_rows,
)
from .decomp import Subdomain, TwoLevelDecomposition, build_two_level
from .errors import (
    ConfigError,
    DeviceError,
    EigensolveError,
    ModeCapError,
    NearResonanceError,
    NoConvergenceError,
    SingularOperatorError,
    SolverError,
)
from .fem import (
    AssembledForms,
    CoefficientField,
    FeSpace,
    Mesh,
    assemble_forms,
    assemble_local_forms,
    assemble_rhs,
    build_fe_space,
    build_unit_square_mesh,
    coefficient_field,
    loguniform_cell_field,
    triangle_areas,
)
from .problems import CONFIGS, Problem, ProblemConfig, build_problem, estimate_cstab_sparse
from .schwarz import (
    CsrOperator,
    DeviceOperator,
    LocalSolver,
    TwoLevelPreconditioner,
    factorize,
)
from .wgmres import GmresReport, elman_gamma, weighted_gmres, weighted_gmres_batch
from .analysis import CheckReport, check_prop26_identity, check_t0_stability, check_tf_stability, fov_bounds

__version__ = "0.1.0"
