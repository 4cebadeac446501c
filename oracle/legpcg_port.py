"""ORACLE -- CPU restatement of the reference legpcg hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2004_13961_b200`` imports this
module; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may, and only as the checker or
as the timed CPU baseline -- never as the product path.

Each function restates one reference function (file:line relative to
``/root/reference``).  The dense parts use numpy (OpenBLAS dgemm, as the
reference does); the sequential sparse kernels are the plain-C port in
``oracle/ilu_port.c``.  One deliberate deviation, the one SURVEY.md section 0.2
prescribes: the preconditioner solve is ILU(0) for every dimension (the
reference's own 1-D branch, ``pcg.py:92-94``), not its d >= 2 LAPACK
banded-Cholesky substitution.

Parity pin: ``tests/golden/make_golden.py`` runs the real reference (imported
read-only in the build container) on seeded inputs and commits the outputs
under ``tests/golden/``; ``tests/test_oracle_golden.py`` checks this port
against them (bitwise for the quadrature rule, the Legendre table and the
ILU(0) factors; to rounding for everything built from BLAS products).
"""

from __future__ import annotations

import ctypes
import itertools
import os
import time

import numpy as np
import scipy.sparse as sp

_HERE = os.path.dirname(os.path.abspath(__file__))


# ---------------------------------------------------------------------------
# L1: Legendre kernel (reference pkg/src/legpcg/legendre.py)
# ---------------------------------------------------------------------------

def legendre_table(x, nmax):
    """T[j, n] = L_n(x_j) by the three-term recurrence (legendre.py:86-95)."""
    x = np.asarray(x, dtype=float)
    t = np.empty((x.size, nmax + 1))
    t[:, 0] = 1.0
    if nmax >= 1:
        t[:, 1] = x
    for k in range(1, nmax):
        t[:, k + 1] = ((2 * k + 1) * x * t[:, k] - k * t[:, k - 1]) / (k + 1)
    return t


def _pn_dpn(n, x):
    """L_n and L_n' (legendre.py:98-106)."""
    prev, cur = np.ones_like(x), x.copy()
    for k in range(1, n):
        prev, cur = cur, ((2 * k + 1) * x * cur - k * prev) / (k + 1)
    return cur, n * (prev - x * cur) / (1.0 - x * x)


def gauss_rule(order, tol=1e-15, max_iter=100):
    """(nodes, weights) of the order-P Gauss rule (legendre.py:109-145)."""
    n = int(order)
    if n == 1:
        return np.array([0.0]), np.array([2.0])
    x = np.cos(np.pi * (4 * np.arange(n) + 3) / (4 * n + 2))
    for _ in range(max_iter):
        p, dp = _pn_dpn(n, x)
        step = p / dp
        x -= step
        if np.max(np.abs(step)) < tol:
            break
    else:
        raise RuntimeError("Gauss-Newton did not converge")
    p, dp = _pn_dpn(n, x)
    x -= p / dp
    x = x[::-1].copy()
    x = 0.5 * (x - x[::-1])
    _, dp = _pn_dpn(n, x)
    w = 2.0 / ((1.0 - x * x) * dp * dp)
    w = 0.5 * (w + w[::-1])
    return x, w


def phi_to_legendre(u, axis):
    """out_k = u_k - u_{k-2}, K -> K+2 along ``axis`` (legendre.py:176-194)."""
    u = np.moveaxis(np.asarray(u, dtype=float), axis, 0)
    out = np.zeros((u.shape[0] + 2,) + u.shape[1:])
    out[:-2] += u
    out[2:] -= u
    return np.moveaxis(out, 0, axis)


def dphi_to_legendre(u, axis):
    """out_{k+1} = -(2k+3) u_k, K -> K+2 (legendre.py:197-215)."""
    u = np.moveaxis(np.asarray(u, dtype=float), axis, 0)
    k = u.shape[0]
    out = np.zeros((k + 2,) + u.shape[1:])
    coef = -(2.0 * np.arange(k) + 3.0).reshape((k,) + (1,) * (u.ndim - 1))
    out[1:k + 1] = coef * u
    return np.moveaxis(out, 0, axis)


# ---------------------------------------------------------------------------
# L2: dense ("reference" mode) transforms (transforms.py:289-375)
# ---------------------------------------------------------------------------

class Plan:
    """TransformPlan in reference mode (transforms.py:298-325)."""

    def __init__(self, order):
        self.order = int(order)
        self.nodes, self.weights = gauss_rule(self.order)
        self.table = legendre_table(self.nodes, self.order - 1)
        self.scale = (2.0 * np.arange(self.order) + 1.0) / 2.0

    def bdlt2(self, c):
        return self.table @ c

    def fdlt2(self, f):
        return self.scale[:, None] * (self.table.T @ (self.weights[:, None] * f))


def _axiswise(worker, a):
    """_axis_apply/_tensor (transforms.py:348-365): axis 0 first."""
    a = np.asarray(a, dtype=float)
    for ax in range(a.ndim):
        m = np.moveaxis(a, ax, 0)
        shp = m.shape
        res = worker(np.ascontiguousarray(m.reshape(shp[0], -1)))
        a = np.moveaxis(res.reshape(shp), 0, ax)
    return a


def tensor_bdlt(plan, c):
    return _axiswise(plan.bdlt2, c)


def tensor_fdlt(plan, f):
    return _axiswise(plan.fdlt2, f)


# ---------------------------------------------------------------------------
# L3: matrix-free operator (operator.py:95-222)
# ---------------------------------------------------------------------------

def mass_contract(v, axis):
    """out_k = 2v_k/(2k+1) - 2v_{k+2}/(2k+5) (operator.py:131-144)."""
    m = np.moveaxis(v, axis, 0)
    k = m.shape[0] - 2
    ks = np.arange(k, dtype=float).reshape((k,) + (1,) * (m.ndim - 1))
    out = (2.0 / (2 * ks + 1)) * m[:k] - (2.0 / (2 * ks + 5)) * m[2:]
    return np.moveaxis(out, 0, axis)


def stiff_contract(v, axis):
    """out_k = -2 v_{k+1} (operator.py:147-152)."""
    m = np.moveaxis(v, axis, 0)
    return np.moveaxis(-2.0 * m[1:-1], 0, axis)


def grid(spec, plan, role):
    """Coefficient values on the tensor Gauss grid (operator.py:95-120)."""
    if isinstance(role, tuple):   # ('axis_beta', i): 1-D field along axis i
        i = role[1]
        vals = spec.axis_betas[i](plan.nodes)
        shape = [1] * spec.dim
        shape[i] = plan.order
        return vals.reshape(shape)
    fld = {"beta": spec.beta, "alpha": spec.alpha, "rhs": spec.rhs}[role]
    return fld.on_grid([plan.nodes] * spec.dim)


def _diffusion(spec, plan, i, cache):
    role = ("axis_beta", i) if spec.axis_betas is not None else "beta"
    if role not in cache:
        cache[role] = grid(spec, plan, role)
        if np.min(cache[role]) <= 0.0:
            raise ValueError("diffusion coefficient is not positive on the grid")
    return cache[role]


def apply_A(spec, plan, u, cache=None):
    """(operator.py:161-174); u is the K^d tensor with axis 0 = x."""
    cache = {} if cache is None else cache
    d = spec.dim
    out = np.zeros_like(u)
    for i in range(d):
        g = u
        for a in range(d):
            g = dphi_to_legendre(g, a) if a == i else phi_to_legendre(g, a)
        g = tensor_bdlt(plan, g) * _diffusion(spec, plan, i, cache)
        h = tensor_fdlt(plan, g)
        for a in range(d):
            h = stiff_contract(h, a) if a == i else mass_contract(h, a)
        out += h
    return out


def apply_B(spec, plan, u, cache=None):
    """(operator.py:177-187)."""
    cache = {} if cache is None else cache
    if spec.alpha is None or spec.alpha.is_zero:
        return np.zeros_like(u)
    if "alpha" not in cache:
        cache["alpha"] = grid(spec, plan, "alpha")
    g = u
    for a in range(spec.dim):
        g = phi_to_legendre(g, a)
    h = tensor_fdlt(plan, tensor_bdlt(plan, g) * cache["alpha"])
    for a in range(spec.dim):
        h = mass_contract(h, a)
    return h


def apply_system(spec, plan, u, cache=None):
    """(A + B) u (operator.py:204-210)."""
    cache = {} if cache is None else cache
    out = apply_A(spec, plan, u, cache)
    if spec.alpha is not None and not spec.alpha.is_zero:
        out += apply_B(spec, plan, u, cache)
    return out


def assemble_rhs(spec, plan):
    """F_k = (I_N f, phi_k) (operator.py:213-222)."""
    h = tensor_fdlt(plan, grid(spec, plan, "rhs"))
    for a in range(spec.dim):
        h = mass_contract(h, a)
    return h


def rhs_from_legendre(fhat):
    """F = per-axis mass contraction of a P^d Legendre series."""
    h = np.asarray(fhat, dtype=float)
    for a in range(h.ndim):
        h = mass_contract(h, a)
    return h


# ---------------------------------------------------------------------------
# L3: preconditioner assembly (precond.py:75-297)
# ---------------------------------------------------------------------------

def expand_coefficient(field, t, dim):
    """Degree-t Legendre truncation of a field (precond.py:75-87)."""
    plan = Plan(max(2 * (t + 1), 32))
    hat = tensor_fdlt(plan, field.on_grid([plan.nodes] * dim))
    return hat[(slice(0, t + 1),) * dim].copy()


def _block_offsets(kind, t):
    reach = t if kind == "stiff" else t + 2
    return [o for o in range(-reach, reach + 1) if (o - t) % 2 == 0]


def building_blocks_1d(T, K, nodes, weights):
    """Diagonals of S^(t)[i,m] = (L_t phi_i', phi_m'), M^(t) = (L_t phi_i, phi_m)
    by exact Gauss quadrature (precond.py:118-161).  Returns two lists (over t)
    of dicts offset -> length-K diagonal (entry i holds (i, i+o))."""
    Q = nodes.size
    acc = {kind: [{o: np.zeros(K) for o in _block_offsets(kind, t)}
                  for t in range(T + 1)] for kind in ("stiff", "mass")}
    dcoef = -(2.0 * np.arange(K) + 3.0)
    for lo in range(0, Q, 512):
        hi = min(lo + 512, Q)
        tab = legendre_table(nodes[lo:hi], K + 1)
        basis = {"mass": tab[:, :K] - tab[:, 2:K + 2],
                 "stiff": dcoef * tab[:, 1:K + 1]}
        w = weights[lo:hi]
        for t in range(T + 1):
            wt = w * tab[:, t]
            for kind in ("stiff", "mass"):
                b = basis[kind]
                for o, diag in acc[kind][t].items():
                    if o >= 0:
                        diag[:K - o] += np.einsum("p,pi,pi->i", wt, b[:, :K - o], b[:, o:])
    for kind in ("stiff", "mass"):
        for t in range(T + 1):
            for o, diag in acc[kind][t].items():
                if o < 0:
                    diag[-o:] = acc[kind][t][-o][:K + o]
    return acc["stiff"], acc["mass"]


def hat_groups(spec, t1, t2):
    """(hat, stiff axis) terms (precond.py:175-197)."""
    d = spec.dim
    groups = []
    if spec.axis_betas is not None:
        cuts = t1 if isinstance(t1, (tuple, list)) else (t1,) * d
        for i in range(d):
            h1 = expand_coefficient(spec.axis_betas[i], cuts[i], 1)
            shape = [1] * d
            shape[i] = cuts[i] + 1
            groups.append((h1.reshape(shape), i))
    else:
        hat = expand_coefficient(spec.beta, int(t1), d)
        groups += [(hat, i) for i in range(d)]
    if spec.alpha is not None and not spec.alpha.is_zero:
        groups.append((expand_coefficient(spec.alpha, int(t2), d), None))
    return groups


_CONTRACT = {1: "a,ai->i", 2: "ab,ai,bj->ij", 3: "abc,ai,bj,cl->ijl"}


def assemble_M(spec, t1, t2):
    """Sparse preconditioner as a scipy CSR matrix, x fastest
    (precond.py:207-248, _symmetrize 255-269, _compress 272-297)."""
    d, K = spec.dim, spec.N - 1
    groups = hat_groups(spec, t1, t2)
    tmax = max(h.shape[a] for h, _ in groups for a in range(d)) - 1
    nodes, weights = gauss_rule(K + tmax // 2 + 2)
    S, M = building_blocks_1d(tmax, K, nodes, weights)
    acc = {}
    for hat, stiff in groups:
        lens = hat.shape
        per_axis = []
        for a in range(d):
            blocks = S if a == stiff else M
            reach = lens[a] - 1 + (0 if a == stiff else 2)
            cand = {}
            for o in range(-reach, reach + 1):
                par = o % 2
                if par >= lens[a]:
                    continue
                stack = np.zeros((lens[a], K))
                for t in range(lens[a]):
                    if o in blocks[t]:
                        stack[t] = blocks[t][o]
                cand[o] = stack[par::2]
            per_axis.append(cand)
        for combo in itertools.product(*[sorted(c) for c in per_axis]):
            sub = hat[tuple(slice(o % 2, None, 2) for o in combo)]
            term = np.einsum(_CONTRACT[d], sub,
                             *[per_axis[a][combo[a]] for a in range(d)],
                             optimize=True)
            if combo in acc:
                acc[combo] += term
            else:
                acc[combo] = term

    def box(c):
        return tuple(slice(max(0, -o), K - max(0, o)) for o in c)

    for combo in {max(c, tuple(-o for o in c)) for c in list(acc)}:
        neg = tuple(-o for o in combo)
        if combo == neg:
            continue
        for key in (combo, neg):
            acc.setdefault(key, np.zeros((K,) * d))
        avg = 0.5 * (acc[combo][box(combo)] + acc[neg][box(neg)])
        acc[combo][box(combo)] = avg
        acc[neg][box(neg)] = avg

    n = K ** d
    stride = np.array([K ** a for a in range(d)], dtype=np.int64)
    rows, cols, vals = [], [], []
    for combo in sorted(acc):
        b = box(combo)
        v = acc[combo][b]
        keep = np.abs(v) >= 1e-300
        if not np.any(keep):
            continue
        g = np.meshgrid(*[np.arange(s.start, s.stop, dtype=np.int64) for s in b],
                        indexing="ij")
        lin = sum(gi * si for gi, si in zip(g, stride))
        shift = int(np.dot(np.array(combo, dtype=np.int64), stride))
        rows.append(lin[keep])
        cols.append(lin[keep] + shift)
        vals.append(v[keep])
    csr = sp.coo_matrix((np.concatenate(vals),
                         (np.concatenate(rows), np.concatenate(cols))),
                        shape=(n, n)).tocsr()
    csr.sort_indices()
    csr.sum_duplicates()
    return csr


# ---------------------------------------------------------------------------
# L3: ILU(0) and the sweeps through the C port (sparse.py:116-221)
# ---------------------------------------------------------------------------

_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "_build", "libilu_port.so")
        if not os.path.exists(path):
            build()
        _LIB = ctypes.CDLL(path)
        p = ctypes.c_void_p
        i64 = ctypes.c_int64
        _LIB.oracle_ilu0.restype = i64
        _LIB.oracle_ilu0.argtypes = [i64, p, p, p, p, ctypes.c_double]
        for name in ("oracle_forward", "oracle_backward", "oracle_spmv"):
            getattr(_LIB, name).restype = None
            getattr(_LIB, name).argtypes = [i64, p, p, p, p, p]
    return _LIB


def build():
    """Compile oracle/ilu_port.c into oracle/_build/ (gcc, -ffp-contract=off)."""
    import subprocess
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


class ZeroPivot(Exception):
    def __init__(self, row):
        self.row = row
        super().__init__(f"zero pivot at elimination step {row}")


class Factors:
    """(L strictly lower, U upper incl. diagonal) as int64 CSR triples."""

    def __init__(self, L, U, n):
        self.L, self.U, self.n = L, U, n


def _csr64(m):
    m = sp.csr_matrix(m)
    m.sort_indices()
    return (m.indptr.astype(np.int64), m.indices.astype(np.int64),
            m.data.astype(float))


def ilu0(m, pivot_tol=1e-300):
    """ILU(0) restricted to NZ(M) (sparse.py:142-172)."""
    indptr, indices, values = _csr64(m)
    n = indptr.size - 1
    diag = np.empty(n, dtype=np.int64)
    for i in range(n):
        lo, hi = indptr[i], indptr[i + 1]
        pos = lo + np.searchsorted(indices[lo:hi], i)
        if pos >= hi or indices[pos] != i:
            raise ZeroPivot(i)
        diag[i] = pos
    data = values.copy()
    bad = _lib().oracle_ilu0(n, _ptr(indptr), _ptr(indices), _ptr(data),
                             _ptr(diag), pivot_tol)
    if bad >= 0:
        raise ZeroPivot(int(bad))
    if abs(data[diag[n - 1]]) < pivot_tol:
        raise ZeroPivot(n - 1)
    lower = np.zeros(indices.size, dtype=bool)
    for i in range(n):
        lower[indptr[i]:diag[i]] = True
    cnt_l = diag - indptr[:-1]
    ip_l = np.concatenate([[0], np.cumsum(cnt_l)]).astype(np.int64)
    ip_u = indptr - ip_l
    L = (ip_l, indices[lower].copy(), data[lower].copy())
    U = (ip_u, indices[~lower].copy(), data[~lower].copy())
    return Factors(L, U, n)


def forward_sub(f, r):
    y = np.zeros(f.n)
    r = np.ascontiguousarray(r, dtype=float)
    _lib().oracle_forward(f.n, *map(_ptr, f.L), _ptr(r), _ptr(y))
    return y


def backward_sub(f, y):
    z = np.zeros(f.n)
    y = np.ascontiguousarray(y, dtype=float)
    _lib().oracle_backward(f.n, *map(_ptr, f.U), _ptr(y), _ptr(z))
    return z


def precond_apply(f, r):
    return backward_sub(f, forward_sub(f, r))


def spmv(m, x):
    indptr, indices, values = _csr64(m)
    y = np.empty(indptr.size - 1)
    x = np.ascontiguousarray(x, dtype=float)
    _lib().oracle_spmv(y.size, _ptr(indptr), _ptr(indices), _ptr(values),
                       _ptr(x), _ptr(y))
    return y


# ---------------------------------------------------------------------------
# L4: PCG (pcg.py:77-179), ILU(0) preconditioner for every d
# ---------------------------------------------------------------------------

def _ldot(a, b):
    """Extended-precision inner product (pcg.py:77-79)."""
    return float(np.dot(a.astype(np.longdouble), b.astype(np.longdouble)))


def pcg_solve(spec, F, epsilon=1e-12, k_max=10_000, preconditioner=None,
              x0=None, timings=None):
    """Returns (x as K^d tensor, dict report).  ``F`` is the K^d tensor
    (axis 0 = x); vectors are x-fastest (Fortran flatten, pcg.py:132-135)."""
    d, K = spec.dim, spec.N - 1
    shape = (K,) * d
    plan = Plan(spec.N + 1)
    cache = {}
    t0 = time.perf_counter()
    psolve = None
    if preconditioner is not None:
        t1, t2 = preconditioner
        fac = ilu0(assemble_M(spec, t1, t2))
        psolve = lambda r: precond_apply(fac, r)  # noqa: E731
    setup = time.perf_counter() - t0

    def op(v):
        u = v.reshape(shape, order="F")
        return apply_system(spec, plan, u, cache).flatten(order="F")

    f = np.asarray(F, dtype=float).flatten(order="F")
    fnorm = float(np.linalg.norm(f))
    x = np.zeros_like(f) if x0 is None else np.asarray(x0, float).flatten(order="F").copy()
    r = f - op(x) if np.any(x) else f.copy()
    hist = [float(np.linalg.norm(r))]
    rho, p, it = 0.0, None, 0
    tl = time.perf_counter()
    while np.sqrt(_ldot(r, r)) > epsilon * fnorm and it < k_max:
        z = psolve(r) if psolve is not None else r
        it += 1
        if it == 1:
            p = z.copy()
            rho = _ldot(r, z)
        else:
            rho_old, rho = rho, _ldot(r, z)
            p = z + (rho / rho_old) * p
        w = op(p)
        curv = _ldot(p, w)
        if curv <= 0.0:
            raise RuntimeError(f"non-positive curvature {curv} at iteration {it}")
        alpha = rho / curv
        x = x + alpha * p
        r = r - alpha * w
        hist.append(float(np.linalg.norm(r)))
    loop = time.perf_counter() - tl
    if timings is not None:
        timings.update(setup_s=setup, loop_s=loop)
    rep = {"iterations": it,
           "converged": bool(np.sqrt(_ldot(r, r)) <= epsilon * fnorm),
           "final_relative_residual": float(np.linalg.norm(r)) / fnorm if fnorm > 0 else 0.0,
           "residual_history": np.array(hist)}
    return x.reshape(shape, order="F"), rep
