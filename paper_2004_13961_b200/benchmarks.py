"""Paper-table benchmark runs on the GPU path (pcg.py:182-271 of the reference).

``BENCHMARKS`` holds, per example, the tabulated N values, the (t1, t2)
truncation pairs and the stopping tolerance (the reference's calibrated
values, ``pcg.py:188-214``); ``make_problem``, ``benchmark_rhs`` and
``run_benchmark`` keep the reference signatures and row format.  The
difference is the one of ``pcg_solve``: the preconditioner is the paper's
one-sweep ILU(0) for every dimension (the reference substitutes a banded
Cholesky solve for d >= 2), so iteration counts are those of ILU(0)-PCG,
including PCG-I (t = 0).  ``transform_mode`` is accepted for compatibility;
every mode runs the dense DMMA transforms.
"""

from __future__ import annotations

import numpy as np

from .coefficients import preset
from .operator import ProblemSpec, SpectralCoeffs
from .pcg import SolverConfig, pcg_solve
from .transforms import TransformPlan

__all__ = ["BENCHMARKS", "make_problem", "benchmark_rhs", "run_benchmark"]

_N1 = [320, 640, 1280, 2560, 5120, 10240]
_N2 = [40, 60, 80, 100, 120]
_N3 = [12, 16, 20, 24]

BENCHMARKS = {
    "example1a": {"N_list": _N1, "t_pairs": [(0, 0), (4, 2), (6, 2)], "epsilon": 1e-10},
    "example1b": {"N_list": _N1, "t_pairs": [(0, 0), (4, 0), (5, 0)], "epsilon": 1e-10},
    "example2a": {"N_list": _N2, "t_pairs": [(0, 0), (4, 3), (6, 3)], "epsilon": 1e-7},
    "example2b": {"N_list": _N2, "t_pairs": [(0, 0), (5, 0), (7, 0)], "epsilon": 1e-10},
    "example3a": {"N_list": _N3, "t_pairs": [(0, 0), (4, 3), (6, 3)], "epsilon": 1e-7},
    "example3b": {"N_list": _N3, "t_pairs": [(0, 0), (5, 0), (6, 0)], "epsilon": 1e-9},
    "example4a": {"N_list": _N2, "t_pairs": [((0, 0), 0), ((4, 3), 0), ((5, 3), 0)],
                  "epsilon": 1e-13},
    "example4b": {"N_list": _N3, "t_pairs": [((0, 0, 0), 0), ((4, 3, 3), 0), ((6, 3, 3), 0)],
                  "epsilon": 1e-13},
}


def make_problem(case, n):
    """ProblemSpec of a named example at N = n (pcg.py:217-221)."""
    p = preset(case)
    return ProblemSpec(dim=p["dim"], N=n, beta=p["beta"], alpha=p["alpha"],
                       axis_betas=p["axis_betas"])


def benchmark_rhs(spec, seed=None):
    """All-ones coefficients, or a seeded Philox normal vector (pcg.py:224-231)."""
    shape = (spec.n_modes,) * spec.dim
    if seed is None:
        return SpectralCoeffs(np.ones(shape))
    return SpectralCoeffs(np.random.Generator(np.random.Philox(seed)).standard_normal(shape))


def run_benchmark(case, n_list=None, t_pairs=None, config=None, seed=None,
                  transform_mode=None):
    """One GPU ILU(0)-PCG solve per (t1, t2, N) cell; rows in table order."""
    if case not in BENCHMARKS:
        raise KeyError(f"unknown benchmark case {case!r}")
    defaults = BENCHMARKS[case]
    n_list = defaults["N_list"] if n_list is None else list(n_list)
    t_pairs = defaults["t_pairs"] if t_pairs is None else list(t_pairs)
    if not n_list:
        raise ValueError("empty N list")
    base = config or SolverConfig(epsilon=defaults["epsilon"])
    rows = []
    for t1, t2 in t_pairs:
        for n in n_list:
            spec = make_problem(case, n)
            plan = TransformPlan(n + 1, mode=transform_mode or "reference")
            cfg = SolverConfig(epsilon=base.epsilon, k_max=base.k_max, preconditioner=(t1, t2),
                               record_history=base.record_history)
            _, rep = pcg_solve(spec, cfg, plan, benchmark_rhs(spec, seed))
            rows.append({"example": case, "d": spec.dim, "N": n, "t1": t1, "t2": t2,
                         "iterations": rep.iterations, "converged": rep.converged,
                         "rel_residual": rep.final_relative_residual,
                         "setup_s": rep.setup_seconds, "iter_mean_s": rep.iter_seconds_mean})
    return rows
