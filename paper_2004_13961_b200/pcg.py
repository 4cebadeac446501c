"""Preconditioned CG on the GPU (drop-in for pcg.py:24-179).

``pcg_solve`` keeps the reference signature and report.  Setup assembles M
on the device and factors it with ILU(0) -- for every dimension, as the paper
and SURVEY.md section 0.2 prescribe (the reference substitutes a banded Cholesky solve
for d >= 2).  The loop (``lp_pcg_solve``, csrc/pcg.cu) keeps every vector on
the device; per iteration it runs the two sweeps, the matvec passes and the
fused update/dot kernels, and reads back one status block for the stopping
test and the curvature check.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib, device
from .operator import SpectralCoeffs
from .precond import assemble_M
from .sparse import ilu0

__all__ = ["SolverConfig", "SolveReport", "IndefiniteOperatorError", "pcg_solve",
           "pcg_solve_device", "setup_preconditioner"]


class IndefiniteOperatorError(RuntimeError):
    """p'Ap <= 0 encountered (pcg.py:34-42)."""

    def __init__(self, iteration, value):
        self.iteration = iteration
        self.value = value
        super().__init__(f"non-positive curvature p'Ap = {value:.3e} at iteration {iteration}")


@dataclass(frozen=True)
class SolverConfig:
    epsilon: float = 1e-12
    k_max: int = 10_000
    preconditioner: Optional[tuple] = None
    record_history: bool = True

    def __post_init__(self):
        if not self.epsilon > 0:
            raise ValueError("epsilon must be positive")
        if self.k_max < 1:
            raise ValueError("k_max must be at least 1")


@dataclass
class SolveReport:
    iterations: int
    converged: bool
    final_relative_residual: float
    residual_history: Optional[np.ndarray]
    setup_seconds: float
    iter_seconds_mean: float
    config: dict = field(default_factory=dict)
    kernel_launches: int = 0


def setup_preconditioner(spec, config, plan):
    """assemble_M + ilu0 on the device; returns the factors (or None)."""
    if config.preconditioner is None:
        return None
    t1, t2 = config.preconditioner
    return ilu0(assemble_M(spec, t1, t2, plan))


def pcg_solve_device(spec, config, plan, f_flat, x_flat=None, factors=None):
    """Device-level solve: f_flat (CUDA, x fastest) -> (x_flat, report dict).

    ``factors`` may be passed to reuse a factored preconditioner."""
    spec._check_plan(plan)
    lib = _lib.load()
    n = spec.n_modes ** spec.dim
    op = spec.device_operator(plan)
    if factors is None:
        factors = setup_preconditioner(spec, config, plan)
    has_x0 = x_flat is not None
    x = x_flat.clone() if has_x0 else device.empty(n)
    hist = np.zeros(config.k_max + 1) if config.record_history else None
    rep = _lib.LpReport()
    rc = lib.lp_pcg_solve(op, factors._handle if factors is not None else None,
                          f_flat.data_ptr(), x.data_ptr(), int(has_x0), config.epsilon,
                          config.k_max, hist.ctypes.data if hist is not None else None,
                          ctypes.byref(rep), _lib.stream_ptr())
    if rc == _lib.LP_ERR_INDEFINITE:
        raise IndefiniteOperatorError(int(rep.iterations), float(rep.indefinite_value))
    _lib.check(rc, "pcg_solve")
    it = int(rep.iterations)
    return x, {"iterations": it, "converged": bool(rep.converged),
               "final_relative_residual": float(rep.final_relative_residual),
               "residual_history": hist[:it + 1].copy() if hist is not None else None,
               "loop_seconds": float(rep.loop_seconds),
               "kernel_launches": int(rep.kernel_launches)}


def pcg_solve(spec, config, plan, F, x0=None):
    """Conjugate gradient on (A+B)x = F with one-sweep ILU(0) preconditioning.

    Returns (solution, report); reaching k_max is converged=False, a
    non-positive p'Ap raises IndefiniteOperatorError (pcg.py:111-179)."""
    spec._check_plan(plan)
    d, k = spec.dim, spec.n_modes
    if F.dim != d or F.n_modes != k:
        raise ValueError("right-hand side shape does not match the problem")
    dev_in = device.is_device(F.data)
    t0 = time.perf_counter()
    factors = setup_preconditioner(spec, config, plan)
    spec.device_operator(plan)
    device.torch().cuda.synchronize()
    setup_seconds = time.perf_counter() - t0
    f = device.to_device(device.fortran_flat(F.data))
    x0f = device.to_device(device.fortran_flat(x0.data)) if x0 is not None else None
    x, r = pcg_solve_device(spec, config, plan, f, x0f, factors=factors)
    it = r["iterations"]
    report = SolveReport(
        iterations=it, converged=r["converged"],
        final_relative_residual=r["final_relative_residual"],
        residual_history=r["residual_history"], setup_seconds=setup_seconds,
        iter_seconds_mean=r["loop_seconds"] / it if it else 0.0,
        config={"epsilon": config.epsilon, "k_max": config.k_max,
                "preconditioner": config.preconditioner, "dim": d, "N": spec.N},
        kernel_launches=r["kernel_launches"])
    sol = x if dev_in else device.host(x)
    return SpectralCoeffs(device.from_fortran_flat(sol, k, d)), report
