"""Pin the CPU oracle (oracle/legpcg_port.py + oracle/ilu_port.c) against the
golden vectors the real reference produced (tests/golden/make_golden.py).

Bitwise where the reference's arithmetic is elementwise and deterministic
(Gauss rule, Legendre table, the CSR pattern of M, the ILU(0) factors of the
reference's own M); to rounding where it goes through BLAS."""

import hashlib

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import legpcg_port as op
from paper_2004_13961_b200 import workloads as wl


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def probe(v, seed=99):
    v = np.asarray(v, dtype=float).ravel()
    g = np.random.default_rng(seed).standard_normal(v.size)
    return np.array([v.sum(), np.abs(v).sum(), float(v @ g), float(v @ v)])


def relerr(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    den = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (den if den > 0 else 1.0)


@pytest.mark.parametrize("P", [1, 2, 3, 5, 17, 33, 64, 129, 257, 513, 2049])
def test_gauss_rule_bitwise(golden, P):
    g = golden("quadrature")
    x, w = op.gauss_rule(P)
    np.testing.assert_array_equal(x, g[f"gauss{P}_nodes"])
    np.testing.assert_array_equal(w, g[f"gauss{P}_weights"])


def test_gauss_rule_known_answers():
    # reference tests/test_legendre.py:65-78 (orders 2 and 3)
    x, w = op.gauss_rule(2)
    np.testing.assert_allclose(x, [-1 / np.sqrt(3), 1 / np.sqrt(3)], atol=1e-15)
    np.testing.assert_allclose(w, [1.0, 1.0], atol=1e-15)
    x, w = op.gauss_rule(3)
    np.testing.assert_allclose(x, [-np.sqrt(0.6), 0.0, np.sqrt(0.6)], atol=1e-15)
    np.testing.assert_allclose(w, [5 / 9, 8 / 9, 5 / 9], atol=1e-15)


@pytest.mark.parametrize("P", [129, 257, 513, 2049])
def test_legendre_table_bitwise(golden, P):
    g = golden("quadrature")
    x, _ = op.gauss_rule(P)
    assert sha(op.legendre_table(x, P - 1)) == str(g[f"table{P}_sha"])


def test_legendre_table33(golden):
    g = golden("quadrature")
    np.testing.assert_array_equal(op.legendre_table(g["gauss33_nodes"], 32), g["table33"])


@pytest.mark.parametrize("d,P", [(1, 33), (2, 17), (3, 9), (2, 129)])
def test_transforms(golden, d, P):
    g = golden("transforms")
    plan = op.Plan(P)
    k = f"tr{d}d{P}"
    assert relerr(op.tensor_bdlt(plan, g[k + "_c"]), g[k + "_bdlt"]) < 1e-14
    assert relerr(op.tensor_fdlt(plan, g[k + "_f"]), g[k + "_fdlt"]) < 1e-14


def _spec(w, N):
    from types import SimpleNamespace
    return SimpleNamespace(dim=w.dim, N=N, beta=w.beta, alpha=w.alpha,
                           rhs=w.rhs_field, axis_betas=None)


@pytest.mark.parametrize("name,N", [("cfg1", 16), ("cfg1", 128), ("cfg2", 24), ("cfg2", 256),
                                    ("cfg3", 64), ("cfg4", 10), ("cfg4", 24), ("cfg5", 12)])
def test_matvec(golden, name, N):
    g = golden("matvec")
    w = wl.CONFIGS[name]()
    spec = _spec(w, N)
    plan = op.Plan(N + 1)
    u = np.random.default_rng(7).standard_normal((N - 1,) * w.dim)
    k = f"mv_{name}_N{N}"
    assert relerr(op.apply_A(spec, plan, u), g[k + "_A"]) < 1e-14
    assert relerr(op.apply_B(spec, plan, u), g[k + "_B"]) < 1e-14
    assert relerr(op.apply_system(spec, plan, u), g[k + "_sys"]) < 1e-14


def test_matvec_axis_betas(golden):
    from types import SimpleNamespace
    from paper_2004_13961_b200.coefficients import CoefficientField
    ab = (CoefficientField(1, lambda x: np.exp(2 * x), "e2x"),
          CoefficientField(1, np.cos, "cosx"), CoefficientField(1, np.cos, "cosx"))
    spec = SimpleNamespace(dim=3, N=8, beta=None, axis_betas=ab, rhs=None,
                           alpha=CoefficientField(3, lambda x, y, z: 1 + x * x, "1+x2"))
    u = np.random.default_rng(8).standard_normal((7, 7, 7))
    out = op.apply_system(spec, op.Plan(9), u)
    assert relerr(out, golden("matvec")["mv_axisbeta3d_N8_sys"]) < 1e-14


PRECOND = [("cfg1", 32, 8), ("cfg2", 16, 4), ("cfg2", 20, 10), ("cfg3", 20, 12),
           ("cfg4", 10, 2), ("cfg4", 12, 8), ("cfg5", 12, 3)]


@pytest.mark.parametrize("name,N,T", PRECOND)
def test_assemble_ilu_sweeps(golden, name, N, T):
    g = golden("precond")
    w = wl.CONFIGS[name]()
    k = f"pc_{name}_N{N}_T{T}"
    m = op.assemble_M(_spec(w, N), T, T)
    assert m.nnz == int(g[k + "_nnz"])
    assert sha(m.indptr.astype(np.int64), m.indices.astype(np.int64)) == str(g[k + "_pattern_sha"])
    np.testing.assert_allclose(probe(m.data), g[k + "_values_probe"], rtol=1e-12)
    # ILU(0) of the reference's own M is bit-identical when M is stored
    if k + "_values" in g:
        mref = sp.csr_matrix((g[k + "_values"], g[k + "_indices"], g[k + "_indptr"]),
                             shape=m.shape)
        fac = op.ilu0(mref)
        assert sha(fac.L[2]) == str(g[k + "_L_sha"])
        assert sha(fac.U[2]) == str(g[k + "_U_sha"])
        np.testing.assert_array_equal(op.forward_sub(fac, g[k + "_r"]), g[k + "_fwd"])
        np.testing.assert_array_equal(op.precond_apply(fac, g[k + "_r"]), g[k + "_z"])
    else:
        fac = op.ilu0(m)
        np.testing.assert_allclose(probe(fac.L[2]), g[k + "_L_probe"], rtol=1e-9)
        np.testing.assert_allclose(probe(fac.U[2]), g[k + "_U_probe"], rtol=1e-9)
        assert relerr(op.precond_apply(fac, g[k + "_r"]), g[k + "_z"]) < 1e-11


@pytest.mark.parametrize("name,N,T", [("cfg1", 128, 8), ("cfg2", 32, 10), ("cfg3", 64, 12),
                                      ("cfg4", 12, 8), ("cfg5", 16, 8)])
def test_pcg(golden, name, N, T):
    g = golden("pcg")
    w = wl.CONFIGS[name]()
    k = f"pcg_{name}_N{N}_T{T}"
    x, rep = op.pcg_solve(_spec(w, N), g[k + "_F"], epsilon=w.rtol, preconditioner=(T, T))
    assert abs(rep["iterations"] - int(g[k + "_iters"])) <= 0
    assert relerr(x, g[k + "_x"]) < 1e-12
    np.testing.assert_allclose(rep["residual_history"], g[k + "_hist"], rtol=1e-6)


def test_cfg1_rhs_and_accuracy(golden):
    """cfg 1: F = assemble_rhs of the manufactured f; the solution is
    spectrally accurate (L2 error ~1e-13)."""
    g = golden("pcg")
    w = wl.cfg1()
    spec = _spec(w, 128)
    F = op.assemble_rhs(spec, op.Plan(129))
    assert relerr(F, g["pcg_cfg1_N128_T8_F"]) < 1e-14
    x = g["pcg_cfg1_N128_T8_x"]
    plan = op.Plan(129)
    uh = op.phi_to_legendre(x, 0)
    vals = plan.table @ uh
    err = np.sqrt(np.sum(plan.weights * (vals - wl.manufactured_solution_1d()(plan.nodes)) ** 2))
    assert err < 1e-12


@pytest.mark.parametrize("name,N,T", [("cfg4", 10, 2), ("cfg5", 9, 1)])
def test_ilu_3d_reference_M_bitwise(golden, name, N, T):
    """3-D: the C port's ILU(0) of the reference's own M is bit-identical to the
    reference's factors; its sweeps equal the reference's."""
    g = golden("large")
    k = f"lpc_{name}_N{N}_T{T}"
    n = g[k + "_indptr"].size - 1
    mref = sp.csr_matrix((g[k + "_values"], g[k + "_indices"], g[k + "_indptr"]), shape=(n, n))
    fac = op.ilu0(mref)
    assert sha(fac.L[2]) == str(g[k + "_L_sha"])
    assert sha(fac.U[2]) == str(g[k + "_U_sha"])
    np.testing.assert_array_equal(op.precond_apply(fac, g[k + "_r"]), g[k + "_z"])


@pytest.mark.parametrize("d,P", [(2, 257), (2, 513), (1, 2049)])
def test_transforms_large(golden, d, P):
    g = golden("large")
    rng = np.random.default_rng(1000 + P + d)
    c = rng.standard_normal((P,) * d)
    f = rng.standard_normal((P,) * d)
    plan = op.Plan(P)
    for key, v in ((f"ltr{d}d{P}_bdlt", op.tensor_bdlt(plan, c)),
                   (f"ltr{d}d{P}_fdlt", op.tensor_fdlt(plan, f))):
        assert relerr(np.asarray(v).ravel()[::997], g[key + "_sub"]) < 1e-13
