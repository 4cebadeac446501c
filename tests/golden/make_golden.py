"""Generate the golden vectors that pin the oracle (and, through it, the GPU path).

Runs the REAL reference package read-only from /root/reference (build
container only -- /root/reference does not exist on the GPU box) on the
seeded inputs of paper_2004_13961_b200.workloads and writes small .npz
fixtures next to this script.  The reference's d >= 2 preconditioner solve is
forced onto its own ILU(0) branch (pcg.py:92-94), as SURVEY.md section 0.2 prescribes.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py [group ...]      # default: every group
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import legpcg.pcg as rpcg  # noqa: E402
from legpcg import legendre as rleg  # noqa: E402
from legpcg import operator as rop  # noqa: E402
from legpcg import precond as rpre  # noqa: E402
from legpcg import sparse as rsp  # noqa: E402
from legpcg import transforms as rtr  # noqa: E402

from paper_2004_13961_b200 import workloads as wl  # noqa: E402
from paper_2004_13961_b200.coefficients import CoefficientField  # noqa: E402


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def probe(v, seed=99):
    """Order-sensitive scalar summaries of a long vector."""
    v = np.asarray(v, dtype=float).ravel()
    g = np.random.default_rng(seed).standard_normal(v.size)
    return np.array([v.sum(), np.abs(v).sum(), float(v @ g), float(v @ v)])


def ref_spec(w, N=None):
    N = w.N if N is None else N
    return rop.ProblemSpec(dim=w.dim, N=N, beta=w.beta, alpha=w.alpha, rhs=w.rhs_field)


def ref_rhs(w, spec, plan):
    if w.rhs_field is not None:
        return rop.assemble_rhs(spec, plan)
    return rop.SpectralCoeffs(wl.mass_contract_series(wl.seeded_fhat(w.dim, spec.N + 1)))


def ilu_everywhere():
    def make(spec, m):
        f = rsp.ilu0(m)
        return lambda r: rsp.precond_apply(f, r)
    rpcg._make_precond_solve = make


def gen_quadrature(out):
    for P in (1, 2, 3, 5, 17, 33, 64, 129, 257, 513, 2049):
        r = rleg.gauss_rule(P)
        out[f"gauss{P}_nodes"] = r.nodes
        out[f"gauss{P}_weights"] = r.weights
    r33 = rleg.gauss_rule(33)
    out["table33"] = rleg.legendre_table(r33.nodes, 32)
    for P in (129, 257, 513, 2049):
        r = rleg.gauss_rule(P)
        out[f"table{P}_sha"] = np.array(sha(rleg.legendre_table(r.nodes, P - 1)))


def gen_transforms(out):
    rng = np.random.default_rng(5)
    for d, P in ((1, 33), (2, 17), (3, 9), (2, 129)):
        plan = rtr.TransformPlan(P)
        c = rng.standard_normal((P,) * d)
        f = rng.standard_normal((P,) * d)
        out[f"tr{d}d{P}_c"] = c
        out[f"tr{d}d{P}_f"] = f
        out[f"tr{d}d{P}_bdlt"] = rtr.tensor_bdlt(plan, c)
        out[f"tr{d}d{P}_fdlt"] = rtr.tensor_fdlt(plan, f)


MATVEC_CASES = [("cfg1", 16), ("cfg1", 128), ("cfg2", 24), ("cfg2", 256),
                ("cfg3", 64), ("cfg4", 10), ("cfg4", 24), ("cfg5", 12)]


def gen_matvec(out):
    for name, N in MATVEC_CASES:
        w = wl.CONFIGS[name]()
        spec = ref_spec(w, N)
        plan = rtr.TransformPlan(N + 1)
        u = np.random.default_rng(7).standard_normal((N - 1,) * w.dim)
        key = f"mv_{name}_N{N}"
        out[key + "_A"] = rop.apply_A(spec, plan, rop.SpectralCoeffs(u)).data
        out[key + "_B"] = rop.apply_B(spec, plan, rop.SpectralCoeffs(u)).data
        out[key + "_sys"] = rop.apply_system(spec, plan, rop.SpectralCoeffs(u)).data
    # axis-separable diffusion form (example 4b shape), 3-D N=8
    ab = (CoefficientField(1, lambda x: np.exp(2 * x), "e2x"),
          CoefficientField(1, np.cos, "cosx"), CoefficientField(1, np.cos, "cosx"))
    spec = rop.ProblemSpec(dim=3, N=8, axis_betas=ab,
                           alpha=CoefficientField(3, lambda x, y, z: 1 + x * x, "1+x2"))
    plan = rtr.TransformPlan(9)
    u = np.random.default_rng(8).standard_normal((7, 7, 7))
    out["mv_axisbeta3d_N8_sys"] = rop.apply_system(spec, plan, rop.SpectralCoeffs(u)).data


PRECOND_CASES = [("cfg1", 32, 8), ("cfg2", 16, 4), ("cfg2", 20, 10),
                 ("cfg3", 20, 12), ("cfg4", 10, 2), ("cfg4", 12, 8), ("cfg5", 12, 3)]


def gen_precond(out):
    for name, N, T in PRECOND_CASES:
        w = wl.CONFIGS[name]()
        spec = ref_spec(w, N)
        plan = rtr.TransformPlan(N + 1)
        m = rpre.assemble_M(spec, T, T, plan)
        key = f"pc_{name}_N{N}_T{T}"
        out[key + "_nnz"] = np.array(m.nnz)
        out[key + "_pattern_sha"] = np.array(sha(m.indptr.astype(np.int64),
                                                 m.indices.astype(np.int64)))
        out[key + "_values_sha"] = np.array(sha(m.values))
        out[key + "_values_probe"] = probe(m.values)
        if m.nnz <= 120_000:
            out[key + "_indptr"] = m.indptr.astype(np.int64)
            out[key + "_indices"] = m.indices.astype(np.int32)
            out[key + "_values"] = m.values
        f = rsp.ilu0(m)
        out[key + "_L_sha"] = np.array(sha(f.L.values))
        out[key + "_U_sha"] = np.array(sha(f.U.values))
        out[key + "_L_probe"] = probe(f.L.values)
        out[key + "_U_probe"] = probe(f.U.values)
        r = np.random.default_rng(11).standard_normal(m.n)
        out[key + "_r"] = r
        out[key + "_fwd"] = rsp.forward_sub(f, r)
        out[key + "_z"] = rsp.precond_apply(f, r)


PCG_CASES = [("cfg1", 128, 8), ("cfg2", 32, 10), ("cfg2", 256, 10), ("cfg3", 64, 12),
             ("cfg4", 12, 8), ("cfg5", 16, 8)]


def gen_pcg(out):
    ilu_everywhere()
    for name, N, T in PCG_CASES:
        w = wl.CONFIGS[name]()
        spec = ref_spec(w, N)
        plan = rtr.TransformPlan(N + 1)
        F = ref_rhs(w, spec, plan)
        cfg = rpcg.SolverConfig(epsilon=w.rtol, preconditioner=(T, T))
        x, rep = rpcg.pcg_solve(spec, cfg, plan, F)
        key = f"pcg_{name}_N{N}_T{T}"
        out[key + "_F"] = F.data
        out[key + "_x"] = x.data
        out[key + "_iters"] = np.array(rep.iterations)
        out[key + "_hist"] = rep.residual_history
        print(key, rep.iterations, rep.final_relative_residual, flush=True)


STRIDE = 997   # subsample stride of the full-size vectors (stored with sha + probes)


def summarise(out, key, v):
    """A vector too large to commit: sha, probes, norm and a strided subsample."""
    v = np.asarray(v, dtype=float).ravel(order="C")
    out[key + "_sha"] = np.array(sha(v))
    out[key + "_probe"] = probe(v)
    out[key + "_sub"] = v[::STRIDE].copy()


LARGE_MATVEC = [("cfg3", 2048), ("cfg4", 128), ("cfg5", 512)]
LARGE_TRANSFORMS = [(2, 257), (2, 513), (2, 2049), (1, 2049), (3, 129)]
LARGE_PRECOND = [("cfg4", 10, 2), ("cfg5", 9, 1)]


def gen_large(out):
    """North-star sizes: full-size matvecs (cfg 3/4/5, C-order K^d inputs from
    default_rng(7)), transforms at P >= 257, and 3-D reference M + factors."""
    for name, N in LARGE_MATVEC:
        w = wl.CONFIGS[name]()
        spec = ref_spec(w, N)
        plan = rtr.TransformPlan(N + 1)
        u = np.random.default_rng(7).standard_normal((N - 1,) * w.dim)
        v = rop.apply_system(spec, plan, rop.SpectralCoeffs(u)).data
        summarise(out, f"lmv_{name}_N{N}", v)
        print("matvec", name, N, flush=True)
    for d, P in LARGE_TRANSFORMS:
        plan = rtr.TransformPlan(P)
        rng = np.random.default_rng(1000 + P + d)
        c = rng.standard_normal((P,) * d)
        f = rng.standard_normal((P,) * d)
        summarise(out, f"ltr{d}d{P}_bdlt", rtr.tensor_bdlt(plan, c))
        summarise(out, f"ltr{d}d{P}_fdlt", rtr.tensor_fdlt(plan, f))
        print("transform", d, P, flush=True)
    for name, N, T in LARGE_PRECOND:
        w = wl.CONFIGS[name]()
        spec = ref_spec(w, N)
        plan = rtr.TransformPlan(N + 1)
        m = rpre.assemble_M(spec, T, T, plan)
        key = f"lpc_{name}_N{N}_T{T}"
        out[key + "_indptr"] = m.indptr.astype(np.int64)
        out[key + "_indices"] = m.indices.astype(np.int32)
        out[key + "_values"] = m.values
        f = rsp.ilu0(m)
        out[key + "_L_sha"] = np.array(sha(f.L.values))
        out[key + "_U_sha"] = np.array(sha(f.U.values))
        r = np.random.default_rng(11).standard_normal(m.n)
        out[key + "_r"] = r
        out[key + "_z"] = rsp.precond_apply(f, r)
        print("precond", key, m.nnz, flush=True)


GROUPS = {"quadrature": gen_quadrature, "transforms": gen_transforms, "matvec": gen_matvec,
          "precond": gen_precond, "pcg": gen_pcg, "large": gen_large}


def main():
    groups = sys.argv[1:] or list(GROUPS)
    for group in groups:
        out = {}
        GROUPS[group](out)
        np.savez_compressed(os.path.join(HERE, f"golden_{group}.npz"), **out)
        print("wrote", group, len(out), "arrays", flush=True)


if __name__ == "__main__":
    main()
