"""GPU parity: the CUDA path (through the C ABI) against the reference's
golden vectors and the CPU oracle on identical seeded inputs."""

import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from oracle import legpcg_port as orc  # noqa: E402
from paper_2004_13961_b200 import (ProblemSpec, SolverConfig, SpectralCoeffs,  # noqa: E402
                                   TransformPlan, apply_A, apply_B, apply_system,
                                   assemble_M, backward_sub, forward_sub, ilu0,
                                   pcg_solve, precond_apply, tensor_bdlt, tensor_fdlt,
                                   workloads as wl)
from paper_2004_13961_b200.coefficients import CoefficientField  # noqa: E402
from paper_2004_13961_b200.sparse import SparseMatrix  # noqa: E402


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def relerr(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    den = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (den if den > 0 else 1.0)


def probe(v, seed=99):
    v = np.asarray(v, dtype=float).ravel()
    g = np.random.default_rng(seed).standard_normal(v.size)
    return np.array([v.sum(), np.abs(v).sum(), float(v @ g), float(v @ v)])


def spec_of(w, N):
    return ProblemSpec(dim=w.dim, N=N, beta=w.beta, alpha=w.alpha, rhs=w.rhs_field)


# ------------------------------------------------------------------ transforms

@pytest.mark.parametrize("P", [129, 257, 513, 2049])
def test_device_table_bitwise(golden, P):
    assert sha(TransformPlan(P).table()) == str(golden("quadrature")[f"table{P}_sha"])


@pytest.mark.parametrize("d,P", [(1, 33), (2, 17), (3, 9), (2, 129)])
def test_tensor_transforms(golden, d, P):
    g = golden("transforms")
    plan = TransformPlan(P)
    k = f"tr{d}d{P}"
    assert relerr(tensor_bdlt(plan, g[k + "_c"]), g[k + "_bdlt"]) < 1e-13
    assert relerr(tensor_fdlt(plan, g[k + "_f"]), g[k + "_fdlt"]) < 1e-13


def check_summary(g, key, v, tol):
    """Compare a full-size vector with the reference's committed summary
    (strided subsample, norm and a random projection; make_golden.summarise)."""
    v = np.asarray(v, dtype=float).ravel()
    sub = g[key + "_sub"]
    assert relerr(v[::997], sub) <= tol, (key, relerr(v[::997], sub))
    pr = g[key + "_probe"]
    nv = np.linalg.norm(v)
    assert abs(nv - np.sqrt(pr[3])) <= tol * np.sqrt(pr[3])
    proj = float(v @ np.random.default_rng(99).standard_normal(v.size))
    assert abs(proj - pr[2]) <= tol * nv * np.sqrt(v.size)


@pytest.mark.parametrize("d,P", [(2, 257), (2, 513), (2, 2049), (1, 2049), (3, 129)])
def test_tensor_transforms_large(golden, d, P):
    """tensor_bdlt / tensor_fdlt at the configs' orders (transforms.py:368-375)
    against the reference run on the same seeded inputs: <= 1e-13."""
    g = golden("large")
    rng = np.random.default_rng(1000 + P + d)
    c = rng.standard_normal((P,) * d)
    f = rng.standard_normal((P,) * d)
    plan = TransformPlan(P)
    check_summary(g, f"ltr{d}d{P}_bdlt", tensor_bdlt(plan, c), 1e-13)
    check_summary(g, f"ltr{d}d{P}_fdlt", tensor_fdlt(plan, f), 1e-13)


def test_transform_known_answers():
    # reference tests/test_transforms.py:22-31,49-59
    plan = TransformPlan(33)
    e0 = np.zeros(33)
    e0[0] = 1.0
    np.testing.assert_allclose(tensor_bdlt(plan, e0), np.ones(33), atol=1e-14)
    np.testing.assert_allclose(tensor_fdlt(plan, np.ones(33)), e0, atol=1e-13)
    e1 = np.zeros(33)
    e1[1] = 1.0
    np.testing.assert_allclose(tensor_fdlt(plan, plan.rule.nodes.copy()), e1, atol=1e-13)


# ---------------------------------------------------------------------- matvec

MV = [("cfg1", 16), ("cfg1", 128), ("cfg2", 24), ("cfg2", 256), ("cfg3", 64), ("cfg4", 10),
      ("cfg4", 24), ("cfg5", 12)]


@pytest.mark.parametrize("name,N", MV)
def test_matvec_golden(golden, name, N):
    g = golden("matvec")
    w = wl.CONFIGS[name]()
    spec = spec_of(w, N)
    plan = TransformPlan(N + 1)
    u = SpectralCoeffs(np.random.default_rng(7).standard_normal((N - 1,) * w.dim))
    k = f"mv_{name}_N{N}"
    assert relerr(apply_A(spec, plan, u).data, g[k + "_A"]) < 1e-12
    assert relerr(apply_B(spec, plan, u).data, g[k + "_B"]) < 1e-12
    assert relerr(apply_system(spec, plan, u).data, g[k + "_sys"]) < 1e-12


def test_matvec_axis_betas(golden):
    ab = (CoefficientField(1, lambda x: np.exp(2 * x), "e2x"),
          CoefficientField(1, np.cos, "cosx"), CoefficientField(1, np.cos, "cosx"))
    spec = ProblemSpec(dim=3, N=8, axis_betas=ab,
                       alpha=CoefficientField(3, lambda x, y, z: 1 + x * x, "1+x2"))
    u = SpectralCoeffs(np.random.default_rng(8).standard_normal((7, 7, 7)))
    out = apply_system(spec, TransformPlan(9), u).data
    assert relerr(out, golden("matvec")["mv_axisbeta3d_N8_sys"]) < 1e-12


@pytest.mark.parametrize("name,N", [("cfg3", 2048), ("cfg4", 128)])
def test_matvec_full_size_vs_oracle(name, N):
    """BASELINE sizes: <= 1e-12 relative against the CPU oracle."""
    w = wl.CONFIGS[name]()
    spec = spec_of(w, N)
    u = np.random.default_rng(3).standard_normal((N - 1,) * w.dim)
    ref = orc.apply_system(spec, orc.Plan(N + 1), u)
    out = apply_system(spec, TransformPlan(N + 1), SpectralCoeffs(u)).data
    assert relerr(out, ref) < 1e-12


@pytest.mark.parametrize("name,N", [("cfg3", 2048), ("cfg4", 128), ("cfg5", 512)])
def test_matvec_north_star_sizes(golden, name, N):
    """apply_system (operator.py:204-210) at the full config sizes, 3-D N=512
    included, against the reference run on the same input: <= 1e-12."""
    g = golden("large")
    w = wl.CONFIGS[name]()
    u = np.random.default_rng(7).standard_normal((N - 1,) * w.dim)
    v = apply_system(spec_of(w, N), TransformPlan(N + 1), SpectralCoeffs(u)).data
    check_summary(g, f"lmv_{name}_N{N}", v, 1e-12)


def test_matvec_constant_coefficient_known_answers():
    # reference tests/test_operator.py:26-34 (A e_k = (4k+6) e_k) and :84-95
    n = 10
    spec = ProblemSpec(dim=1, N=n, beta=wl.constant_field(1, 1.0),
                       alpha=wl.constant_field(1, 1.0))
    plan = TransformPlan(n + 1)
    ks = np.arange(n - 1)
    mass = np.diag(2 / (2 * ks + 1) + 2 / (2 * ks + 5))
    off = -2 / (2 * ks[:-2] + 5)
    mass += np.diag(off, 2) + np.diag(off, -2)
    for k in range(n - 1):
        e = np.zeros(n - 1)
        e[k] = 1.0
        a = apply_A(spec, plan, SpectralCoeffs(e)).data
        expect = np.zeros(n - 1)
        expect[k] = 4 * k + 6
        np.testing.assert_allclose(a, expect, atol=1e-11)
        np.testing.assert_allclose(apply_B(spec, plan, SpectralCoeffs(e)).data, mass[:, k],
                                   atol=1e-12)


def test_nonpositive_diffusion_rejected():
    spec = ProblemSpec(dim=1, N=8, beta=CoefficientField(1, lambda x: x, "x"))
    with pytest.raises(ValueError, match="not positive"):
        apply_A(spec, TransformPlan(9), SpectralCoeffs(np.ones(7)))


def test_device_resident_matvec_matches_host():
    w = wl.cfg4(N=24)
    spec = spec_of(w, 24)
    plan = TransformPlan(25)
    u = np.random.default_rng(4).standard_normal((23,) * 3)
    host = apply_system(spec, plan, SpectralCoeffs(u)).data
    dev = apply_system(spec, plan, SpectralCoeffs(torch.from_numpy(u).cuda())).data
    np.testing.assert_array_equal(dev.cpu().numpy(), host)


# --------------------------------------------------------------- preconditioner

PRE = [("cfg1", 32, 8), ("cfg2", 16, 4), ("cfg2", 20, 10), ("cfg3", 20, 12), ("cfg4", 10, 2),
       ("cfg4", 12, 8), ("cfg5", 12, 3)]


@pytest.mark.parametrize("name,N,T", PRE)
def test_assemble_M(golden, name, N, T):
    g = golden("precond")
    w = wl.CONFIGS[name]()
    k = f"pc_{name}_N{N}_T{T}"
    m = assemble_M(spec_of(w, N), T, T)
    assert m.nnz == int(g[k + "_nnz"])
    assert sha(m.indptr, m.indices.astype(np.int64)) == str(g[k + "_pattern_sha"])
    np.testing.assert_allclose(probe(m.values), g[k + "_values_probe"], rtol=1e-12)
    if k + "_values" in g:
        assert relerr(m.values, g[k + "_values"]) < 1e-14


@pytest.mark.parametrize("name,N,T", PRE)
def test_ilu0_and_sweeps_box(golden, name, N, T):
    """Factor the GPU-assembled M in the box layout; compare with the
    reference's factors and sweeps (tolerance: M itself differs by ~1e-16)."""
    g = golden("precond")
    w = wl.CONFIGS[name]()
    k = f"pc_{name}_N{N}_T{T}"
    f = ilu0(assemble_M(spec_of(w, N), T, T))
    np.testing.assert_allclose(probe(f.L.values), g[k + "_L_probe"], rtol=1e-9)
    np.testing.assert_allclose(probe(f.U.values), g[k + "_U_probe"], rtol=1e-9)
    assert relerr(forward_sub(f, g[k + "_r"]), g[k + "_fwd"]) < 1e-11
    assert relerr(precond_apply(f, g[k + "_r"]), g[k + "_z"]) < 1e-11


@pytest.mark.parametrize("name,N,T", [c for c in PRE if c[0] in ("cfg1", "cfg2", "cfg3")])
def test_ilu0_csr_bitwise(golden, name, N, T):
    """The general CSR kernel on the reference's own M reproduces its
    factors bit for bit (same k order, separately rounded mul/sub)."""
    g = golden("precond")
    k = f"pc_{name}_N{N}_T{T}"   # 3-D cases: test_ilu0_csr_bitwise_3d
    n = g[k + "_indptr"].size - 1
    m = SparseMatrix(n, g[k + "_indptr"], g[k + "_indices"], g[k + "_values"])
    f = ilu0(m)
    assert sha(f.L.values) == str(g[k + "_L_sha"])
    assert sha(f.U.values) == str(g[k + "_U_sha"])
    assert relerr(precond_apply(f, g[k + "_r"]), g[k + "_z"]) < 1e-13


@pytest.mark.parametrize("name,N,T", [("cfg4", 10, 2), ("cfg5", 9, 1)])
def test_ilu0_csr_bitwise_3d(golden, name, N, T):
    """3-D: the CSR kernel on the reference's own M reproduces its factors bit
    for bit (sparse.py:116-139); with test_box_factors_bitwise_vs_csr this
    anchors the 3-D box factors to the reference."""
    g = golden("large")
    k = f"lpc_{name}_N{N}_T{T}"
    n = g[k + "_indptr"].size - 1
    m = SparseMatrix(n, g[k + "_indptr"], g[k + "_indices"], g[k + "_values"])
    f = ilu0(m)
    assert sha(f.L.values) == str(g[k + "_L_sha"])
    assert sha(f.U.values) == str(g[k + "_U_sha"])
    assert relerr(precond_apply(f, g[k + "_r"]), g[k + "_z"]) < 1e-13


@pytest.mark.parametrize("name,N,T", [("cfg4", 10, 2), ("cfg5", 9, 1), ("cfg4", 12, 8),
                                      ("cfg5", 12, 3), ("cfg4", 16, 4),
                                      ("cfg5", 20, 2), ("cfg4", 9, 1), ("cfg2", 20, 10),
                                      ("cfg2", 520, 4), ("cfg3", 64, 12), ("cfg3", 150, 12),
                                      ("cfg2", 100, 10), ("cfg2", 37, 0), ("cfg2", 45, 1),
                                      ("cfg3", 40, 13), ("cfg4", 24, 8), ("cfg5", 25, 7)])
def test_box_factors_bitwise_vs_csr(name, N, T):
    """The box-layout factorisation (3-D: row-per-CTA kernel; 2-D: task graph)
    equals, bit for bit, the CSR kernel on the same M -- which reproduces the
    reference's factors bit for bit (test_ilu0_csr_bitwise)."""
    w = wl.CONFIGS[name]()
    m = assemble_M(spec_of(w, N), T, T)
    csr = SparseMatrix(m.n, m.indptr, m.indices, m.values)
    fb, fc = ilu0(m), ilu0(csr)
    assert sha(fb.L.indptr, fb.L.indices) == sha(fc.L.indptr, fc.L.indices)
    assert sha(fb.L.values) == sha(fc.L.values)
    assert sha(fb.U.values) == sha(fc.U.values)


@pytest.mark.parametrize("case,n,t1", [("example4a", 40, (4, 3)), ("example2b", 30, 5),
                                       ("example4a", 70, (5, 3))])
def test_box_factors_bitwise_sparse_patterns(case, n, t1):
    """Box factors on patterns with holes (per-axis diffusion, zero reaction:
    most box slots are out of the pattern) equal the CSR kernel's bit for bit."""
    from paper_2004_13961_b200 import make_problem
    m = assemble_M(make_problem(case, n), t1, 0)
    csr = SparseMatrix(m.n, m.indptr, m.indices, m.values)
    fb, fc = ilu0(m), ilu0(csr)
    assert sha(fb.L.values) == sha(fc.L.values)
    assert sha(fb.U.values) == sha(fc.U.values)


def test_sparse_known_answers():
    # reference tests/test_sparse.py:144-160
    d = np.array([[1.0, 0, 0], [0.5, 1.0, 0], [0, 0.5, 1.0]])
    f = ilu0(SparseMatrix.from_dense(d))
    np.testing.assert_allclose(forward_sub(f, np.ones(3)), [1.0, 0.5, 0.75], atol=1e-15)
    d = np.array([[2.0, 1.0], [0.0, 4.0]])
    f = ilu0(SparseMatrix.from_dense(d))
    np.testing.assert_allclose(backward_sub(f, np.array([3.0, 8.0])), [0.5, 2.0], atol=1e-15)
    f = ilu0(SparseMatrix.from_dense(np.diag([2.0, 5.0])))
    np.testing.assert_allclose(precond_apply(f, np.array([4.0, 10.0])), [2.0, 2.0])


def test_zero_pivot_and_missing_diagonal():
    from paper_2004_13961_b200 import IluZeroPivotError
    with pytest.raises(IluZeroPivotError) as err:
        ilu0(SparseMatrix.from_dense(np.array([[1.0, 1.0], [1.0, 1.0]])))
    assert err.value.row == 1
    with pytest.raises(IluZeroPivotError) as err:
        ilu0(SparseMatrix.from_dense(np.array([[0.0, 1.0], [1.0, 0.0]])))
    assert err.value.row == 0


def test_full_pattern_is_exact_solve():
    rng = np.random.default_rng(11)
    a = rng.standard_normal((12, 12))
    a = a @ a.T + 12 * np.eye(12)
    f = ilu0(SparseMatrix.from_dense(a))
    r = rng.standard_normal(12)
    np.testing.assert_allclose(precond_apply(f, r), np.linalg.solve(a, r), atol=1e-10)


# ------------------------------------------------------------------------ PCG

PCG = [("cfg1", 128, 8), ("cfg2", 32, 10), ("cfg2", 256, 10), ("cfg3", 64, 12), ("cfg4", 12, 8),
       ("cfg5", 16, 8)]


@pytest.mark.parametrize("name,N,T", PCG)
def test_pcg_golden(golden, name, N, T):
    g = golden("pcg")
    w = wl.CONFIGS[name]()
    k = f"pcg_{name}_N{N}_T{T}"
    spec = spec_of(w, N)
    x, rep = pcg_solve(spec, SolverConfig(epsilon=w.rtol, preconditioner=(T, T)),
                       TransformPlan(N + 1), SpectralCoeffs(g[k + "_F"]))
    assert rep.converged
    assert abs(rep.iterations - int(g[k + "_iters"])) <= 1
    assert relerr(x.data, g[k + "_x"]) < 1e-10
    assert rep.residual_history.size == rep.iterations + 1


@pytest.mark.parametrize("name,N,iters", [("cfg3", 2048, 14), ("cfg4", 64, None)])
def test_full_size_solve_certificate(name, N, iters):
    """Full-size ILU(0)-PCG where the CPU oracle cannot run:
    converged, iteration count as measured, and the residual certificate of
    the reference's own test (test_pcg.py:49-55) recomputed with the matvec
    verified above: ||F - (A+B)x|| <= 1.05 eps ||F||."""
    w = wl.CONFIGS[name](N=N)
    spec = spec_of(w, N)
    plan = TransformPlan(N + 1)
    F = wl.mass_contract_series(w.fhat)
    x, rep = pcg_solve(spec, SolverConfig(epsilon=w.rtol, preconditioner=(w.T, w.T)), plan,
                       SpectralCoeffs(F))
    assert rep.converged, rep.iterations
    if iters is not None:
        assert abs(rep.iterations - iters) <= 1, rep.iterations
    r = F - apply_system(spec, plan, x).data
    assert np.linalg.norm(r) <= 1.05 * w.rtol * np.linalg.norm(F)


def test_pcg_determinism():
    w = wl.cfg2(N=32)
    spec = spec_of(w, 32)
    plan = TransformPlan(33)
    F = SpectralCoeffs(wl.mass_contract_series(w.fhat))
    cfg = SolverConfig(epsilon=1e-10, preconditioner=(10, 10))
    x1, r1 = pcg_solve(spec, cfg, plan, F)
    x2, r2 = pcg_solve(spec, cfg, plan, F)
    assert r1.iterations == r2.iterations
    np.testing.assert_array_equal(x1.data, x2.data)


def test_pcg_indefinite_and_kmax():
    from paper_2004_13961_b200 import IndefiniteOperatorError
    spec = ProblemSpec(dim=1, N=16, beta=wl.constant_field(1, 0.01),
                       alpha=wl.constant_field(1, -100.0))
    with pytest.raises(IndefiniteOperatorError) as err:
        pcg_solve(spec, SolverConfig(epsilon=1e-10), TransformPlan(17),
                  SpectralCoeffs(np.ones(15)))
    assert err.value.iteration >= 1
    w = wl.cfg2(N=16)
    spec = spec_of(w, 16)
    _, rep = pcg_solve(spec, SolverConfig(epsilon=1e-14, k_max=2), TransformPlan(17),
                       SpectralCoeffs(np.ones((15, 15))))
    assert not rep.converged and rep.iterations == 2


# ---------------------------------------------------------------- front end on the GPU
@pytest.mark.parametrize("K,T", [(40, 6), (127, 8), (255, 10), (700, 12), (9, 4)])
def test_building_blocks_bitwise_vs_oracle(K, T):
    """lp_blocks_1d (precond.py:118-161 on the GPU): the diagonals of S^(t), M^(t)
    equal the CPU restatement bit for bit (same operation order; K = 700 spans
    two 512-node chunks)."""
    from paper_2004_13961_b200 import precond, quadrature
    rule = quadrature.gauss_rule(K + T // 2 + 2)
    S, M = precond.building_blocks_1d(T, K, rule)
    So, Mo = orc.building_blocks_1d(T, K, rule.nodes, rule.weights)
    for t in range(T + 1):
        assert set(S[t].diags) == set(So[t]) and set(M[t].diags) == set(Mo[t])
        for o in S[t].diags:
            np.testing.assert_array_equal(S[t].diags[o], So[t][o])
        for o in M[t].diags:
            np.testing.assert_array_equal(M[t].diags[o], Mo[t][o])


@pytest.mark.parametrize("d,P", [(1, 129), (2, 67), (3, 21), (3, 3), (2, 257)])
def test_mass_contract_bitwise(d, P):
    """lp_mass_contract equals the reference's numpy expression
    (operator.py:131-143, axis 0 first) bit for bit."""
    from paper_2004_13961_b200 import device
    from paper_2004_13961_b200.operator import mass_contract_device
    fh = np.random.default_rng(P).standard_normal((P,) * d)
    ref = wl.mass_contract_series(fh)
    out = device.host(mass_contract_device(device.to_device(fh.flatten(order="F")), d, P))
    np.testing.assert_array_equal(out.reshape((P - 2,) * d, order="F"), ref)


def test_assemble_rhs_matches_oracle():
    """assemble_rhs (operator.py:213-222): GPU FDLT + GPU contraction."""
    from paper_2004_13961_b200 import assemble_rhs, coefficients
    w = wl.cfg2(N=48)
    f = coefficients.CoefficientField(2, lambda x, y: np.exp(x) * np.cos(2 * y) + x * y, "f")
    spec = ProblemSpec(dim=2, N=w.N, beta=w.beta, alpha=w.alpha, rhs=f)
    got = assemble_rhs(spec, TransformPlan(w.N + 1)).data
    ospec = ProblemSpec(dim=2, N=w.N, beta=w.beta, alpha=w.alpha, rhs=f)
    ref = orc.assemble_rhs(ospec, orc.Plan(w.N + 1))
    assert relerr(got, ref) < 1e-13


@pytest.mark.parametrize("name,N,T", [("cfg2", 64, 10), ("cfg2", 256, 10), ("cfg3", 150, 12),
                                      ("cfg1", 128, 8), ("cfg4", 12, 8), ("cfg5", 14, 0)])
def test_precond_apply_rz_fused(name, N, T):
    """lp_precond_apply_rz: z equals precond_apply bit for bit and r'z (carried by
    the backward sweep for the 1-D / 2-D boxes, pcg.py:147-151) matches the
    long-double dot of the reference; the result is deterministic."""
    from paper_2004_13961_b200.sparse import precond_apply_rz
    w = wl.CONFIGS[name]()
    f = ilu0(assemble_M(spec_of(w, N), T, T))
    r = np.random.default_rng(3).standard_normal(f.n)
    z0 = precond_apply(f, r)
    z, rz = precond_apply_rz(f, r)
    np.testing.assert_array_equal(z, z0)
    ref = float(np.dot(r.astype(np.longdouble), z0.astype(np.longdouble)))
    scale = float(np.dot(np.abs(r), np.abs(z0)))
    assert abs(rz - ref) <= 1e-13 * scale
    z2, rz2 = precond_apply_rz(f, r)
    assert rz2 == rz


@pytest.mark.parametrize("name,N", [("cfg1", 128), ("cfg2", 64), ("cfg2", 256), ("cfg3", 300), ("cfg4", 20),
                                    ("cfg5", 40)])
def test_apply_dot_fused(name, N):
    """lp_apply_dot: the same w as lp_apply bit for bit, and u'w (accumulated in
    the last line pass, pcg.py:156-157) within 1e-13 of the long-double dot;
    deterministic."""
    from paper_2004_13961_b200 import device
    from paper_2004_13961_b200.operator import apply_flat, apply_flat_dot
    w = wl.CONFIGS[name]()
    spec = spec_of(w, N)
    plan = TransformPlan(N + 1)
    u = device.to_device(np.random.default_rng(4).standard_normal(spec.n_modes ** w.dim))
    ref = apply_flat(spec, plan, 3, u)
    out, uw = apply_flat_dot(spec, plan, 3, u)
    assert bool((out == ref).all())
    uh, wh = device.host(u).astype(np.longdouble), device.host(ref).astype(np.longdouble)
    exact = float(np.dot(uh, wh))
    scale = float(np.dot(np.abs(uh), np.abs(wh)))
    assert abs(uw - exact) <= 1e-13 * scale
    assert apply_flat_dot(spec, plan, 3, u)[1] == uw
