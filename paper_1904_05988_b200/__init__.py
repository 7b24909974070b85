"""B200-native (sm_100a, fp64) hot path of PFASST-SH: spherical-harmonic transforms, the
shallow-water right-hand side, SDC sweeps, two-level FAS transfers and the PFASST block
controller, behind the C ABI in include/pswe.h (libpswe.so). There is no CPU fallback."""
from . import _lib  # noqa: F401
from .transform import (LEGENDRE_RECOMPUTE, LEGENDRE_STREAM, TransformPlan, dealiased_nlon,  # noqa: F401
                        gauss_latitudes, inv_laplacian, laplacian, num_coeffs)
from .swe import ModelParams, SweOde, eval_linear, eval_nonlinear, imex_split, solve_implicit  # noqa: F401
from .sdc import Level, QuadratureTables, build_tables, sdc_run  # noqa: F401
from .multilevel import TransferPair, interpolate_space, mlsdc_step, restrict_space  # noqa: F401
from .pfasst import BlockConfig, Pfasst, run_blocks, schedule  # noqa: F401

__all__ = [
    "TransformPlan", "dealiased_nlon", "gauss_latitudes", "laplacian", "inv_laplacian", "num_coeffs",
    "ModelParams", "SweOde", "eval_linear", "eval_nonlinear", "imex_split", "solve_implicit",
    "Level", "QuadratureTables", "build_tables", "sdc_run",
    "TransferPair", "restrict_space", "interpolate_space", "mlsdc_step",
    "BlockConfig", "Pfasst", "run_blocks", "schedule",
]
