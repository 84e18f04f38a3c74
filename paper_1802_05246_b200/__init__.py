"""B200-native Hermite wave solver hot path (arXiv 1802.05246).

Drop-in for the hot path of the reference package ``hermwave``
(pkg/src/hermwave/__init__.py): grid/field types, scheme and boundary
configuration, the staggered half-step advance of the dissipative and
conservative schemes, and the L2 error diagnostics — with the arithmetic in
hand-written sm_100a kernels behind the C ABI of include/hermb200.h.
"""

from .config import BoundarySpec, BoundarySpec2D, SchemeConfig
from .fields import DUAL, PRIMAL, Field1D, Field2D, FieldPair, Grid1D, Grid2D, TwoLevelState, flip
from .initdata import (
    data_on_grid_1d,
    gaussian_box_u,
    gaussian_box_v,
    gaussian_derivs,
    planewave_on_grid,
    scale_cols,
    sine_derivs,
    standing_wave_on_grid,
)
from .lowlevel import (
    PascalTable,
    apply_interp,
    apply_interp_2d,
    conservative_update_1d,
    conservative_update_2d,
    eval_series,
    expand_taylor,
    expand_taylor_2d,
    ghost_data,
    ghost_data_2d,
    pascal_table,
)
from .norms import (
    ErrorReport,
    PlaneWave2D,
    StandingWave2D,
    conservative_energy,
    conservative_energy_2d,
    default_npts,
    dissipative_energy,
    dissipative_energy_2d,
    fit_rate,
    gauss_rule,
    l2_error_field,
    l2_error_field_2d,
    l2_errors_pair,
)
from .stepping import (
    NumericalError,
    advance_2d,
    advance_conservative,
    bootstrap_first_half,
    full_step_conservative,
    half_step_1d,
    half_step_2d,
    interp_matrix,
    require_finite,
)
from .studies import (
    ConfigError,
    RunConfig,
    make_config,
    parse_config,
    run_conservation_1d,
    run_experiment,
    run_gaussian_1d,
    run_planewave_2d,
)

__version__ = "0.1.0"

__all__ = [
    "BoundarySpec", "BoundarySpec2D", "SchemeConfig",
    "DUAL", "PRIMAL", "Field1D", "Field2D", "FieldPair", "Grid1D", "Grid2D", "TwoLevelState", "flip",
    "planewave_on_grid", "standing_wave_on_grid", "data_on_grid_1d",
    "gaussian_derivs", "gaussian_box_u", "gaussian_box_v", "sine_derivs", "scale_cols",
    "ConfigError", "RunConfig", "make_config", "parse_config", "run_experiment", "run_gaussian_1d",
    "run_conservation_1d", "run_planewave_2d",
    "PascalTable", "apply_interp", "apply_interp_2d", "conservative_update_1d", "conservative_update_2d",
    "eval_series", "expand_taylor", "expand_taylor_2d", "ghost_data", "ghost_data_2d", "pascal_table",
    "ErrorReport", "PlaneWave2D", "StandingWave2D", "default_npts", "fit_rate", "gauss_rule",
    "dissipative_energy", "dissipative_energy_2d", "conservative_energy", "conservative_energy_2d",
    "l2_error_field", "l2_error_field_2d", "l2_errors_pair",
    "NumericalError", "advance_2d", "advance_conservative", "bootstrap_first_half",
    "full_step_conservative", "half_step_1d", "half_step_2d", "interp_matrix", "require_finite",
]
