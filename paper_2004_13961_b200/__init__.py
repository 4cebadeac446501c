"""B200-native (sm_100a, fp64) hot path of the preconditioned Legendre-Galerkin
PCG solver of arXiv:2004.13961, a drop-in for the reference package
``legpcg``'s solver API.  All compute runs in the CUDA library
``_lib/liblegpcg_b200.so`` (C ABI: include/legpcg_b200.h); there is no CPU
fallback.
"""

from .coefficients import (PRESETS, CoefficientField, LegendreSeriesField, constant_field, preset,
                           zero_field)
from .operator import (ProblemSpec, SpectralCoeffs, apply_A, apply_B, apply_system,
                       assemble_rhs)
from .pcg import (IndefiniteOperatorError, SolveReport, SolverConfig, pcg_solve,
                  pcg_solve_device)
from .precond import (BandedBlock, TruncatedCoefficient, assemble_M, building_blocks_1d,
                      expand_coefficient, predicted_bandwidth)
from .quadrature import (GaussRule, dphi_to_legendre, gauss_rule, legendre_table,
                         phi_to_legendre)
from .sparse import (IluFactors, IluZeroPivotError, SparseMatrix, backward_sub, forward_sub,
                     ilu0, precond_apply, spmv)
from .transforms import TransformPlan, bdlt, fdlt, tensor_bdlt, tensor_fdlt
from .benchmarks import BENCHMARKS, benchmark_rhs, make_problem, run_benchmark

__all__ = [n for n in dir() if not n.startswith("_")]
