import sys; sys.path.insert(0,'.')
import numpy as np
from paper_2004_13961_b200 import make_problem, benchmark_rhs, pcg_solve, SolverConfig, TransformPlan, _lib
spec = make_problem("example2a", 40)
F = benchmark_rhs(spec)
for tp in [(4,3), (0,0)]:
    try:
        x, rep = pcg_solve(spec, SolverConfig(epsilon=1e-10, preconditioner=tp), TransformPlan(41), F)
        print(tp, rep.iterations, rep.converged, rep.final_relative_residual)
    except Exception as e:
        import traceback; traceback.print_exc()
