"""B200-native motion-compensated PDHG / SPDHG reconstruction (arXiv 2410.10503).

Drop-in for the hot path of the reference package ``mctomo``: the gated
operators A_i = A o D_i (Joseph ray transform after a rigid / dilatation /
dense warp), step-size selection, and the PDHG / SPDHG solver entry points,
computed by hand-written sm_100a kernels behind a C-ABI
(include/mctomo_b200.h).  There is no CPU fallback.
"""

from .build import build_native
from .experiment_io import (ConvergenceRecord, RasterFormatError, RateFit, fit_rate,
                            load_dataset, load_saddle, read_raster, rmse, save_dataset,
                            save_saddle, write_raster)
from .functionals import fit_value, g_value, moduli, prox_fstar, prox_g
from .linops import (ComposedMap, DiagonalMap, GramSumMap, IdentityMap, LinearMap, StackedMap,
                     adjoint_mismatch, compose, power_method, stacked_norm_sq)
from .motion import DenseWarpOperator, MotionParams, WarpOperator, motion_sequence
from .projector import Geometry, GatedOperator, RayTransform, adjoint, forward, ray_transform
from .simulate import (PHANTOM_KINDS, GatedDataset, NoiseModel, estimate_norms, gate_operators,
                       gaussian_field, gaussian_field_device, generate, make_phantom,
                       nonrigid_preset, rigid_preset, simulate_data)
from .solvers import (RHO, DivergenceError, Problem, SaddlePoint, SolverConfig, SolverState,
                      cg_reference, default_config, draw_sequence, optimality_residual, run,
                      run_batch, sample_gates, step)

__version__ = "0.1.0"
