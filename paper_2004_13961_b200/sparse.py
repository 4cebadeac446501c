"""Sparse matrices, ILU(0) and the triangular sweeps on the GPU
(drop-in for sparse.py:16-232).

A ``SparseMatrix`` is either a host CSR matrix (``from_dense`` /
``from_scipy`` / the constructor, exactly the reference's frozen dataclass
fields) or a device-resident matrix produced by ``assemble_M`` in the
implicit-offset box layout, whose CSR arrays are exported lazily on first
access.  ``ilu0`` / ``forward_sub`` / ``backward_sub`` / ``precond_apply`` /
``spmv`` always run on the GPU (csrc/ilu_csr.cu, csrc/ilu_box.cu).
"""

from __future__ import annotations

import ctypes
import weakref

import numpy as np

from . import _lib, device

__all__ = ["SparseMatrix", "IluFactors", "IluZeroPivotError", "spmv", "ilu0",
           "forward_sub", "backward_sub", "precond_apply", "precond_apply_rz", "save_matrix_market",
           "load_matrix_market"]


class IluZeroPivotError(RuntimeError):
    """Raised when ILU(0) meets a (numerically) zero pivot (sparse.py:30-35)."""

    def __init__(self, row):
        self.row = row
        super().__init__(f"zero pivot at elimination step {row}")


def _destroy(handle):
    try:
        _lib.load(init_device=False).lp_ilu_destroy(handle)
    except Exception:
        pass


class SparseMatrix:
    """CSR matrix with sorted, duplicate-free column indices per row."""

    def __init__(self, n, indptr=None, indices=None, values=None, *, _handle=None, _nnz=None):
        self.n = int(n)
        self._indptr = None if indptr is None else np.asarray(indptr, dtype=np.int64)
        self._indices = None if indices is None else np.asarray(indices)
        self._values = None if values is None else np.asarray(values, dtype=float)
        self._handle = _handle
        self._nnz = _nnz
        if _handle is not None:
            weakref.finalize(self, _destroy, _handle)

    # -- construction ----------------------------------------------------
    @classmethod
    def from_scipy(cls, mat):
        csr = mat.tocsr()
        csr.sort_indices()
        csr.sum_duplicates()
        return cls(csr.shape[0], csr.indptr.astype(np.int64), csr.indices,
                   csr.data.astype(float))

    @classmethod
    def from_dense(cls, dense, tol=0.0):
        import scipy.sparse as sp
        d = np.asarray(dense, dtype=float).copy()
        if tol > 0.0:
            d[np.abs(d) < tol] = 0.0
        return cls.from_scipy(sp.csr_matrix(d))

    # -- CSR arrays (exported from the device for assembled matrices) ----
    def _export(self):
        if self._indptr is None:
            lib = _lib.load()
            nnz = self.nnz
            ip = np.empty(self.n + 1, dtype=np.int64)
            ix = np.empty(nnz, dtype=np.int32)
            v = np.empty(nnz)
            _lib.check(lib.lp_matrix_export(self._handle, 0, ip.ctypes.data, ix.ctypes.data,
                                            v.ctypes.data), "export")
            self._indptr, self._indices, self._values = ip, ix, v

    @property
    def indptr(self):
        self._export()
        return self._indptr

    @property
    def indices(self):
        self._export()
        return self._indices

    @property
    def values(self):
        self._export()
        return self._values

    @property
    def nnz(self):
        if self._indptr is not None:
            return int(self._indptr[-1])
        if self._nnz is None:
            v = ctypes.c_int64()
            _lib.check(_lib.load().lp_matrix_nnz(self._handle, ctypes.byref(v)))
            self._nnz = int(v.value)
        return self._nnz

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.values, self.indices, self.indptr), shape=(self.n, self.n))

    def to_dense(self):
        return self.to_scipy().toarray()

    def validate(self):
        ip, ix = self.indptr, self.indices
        if ip[0] != 0 or ip[-1] != ix.size:
            raise ValueError("inconsistent row pointers")
        if np.any(np.diff(ip) < 0):
            raise ValueError("row pointers must be nondecreasing")
        if ix.size and (ix.min() < 0 or ix.max() >= self.n):
            raise ValueError("column index out of range")
        for i in range(self.n):
            if np.any(np.diff(ix[ip[i]:ip[i + 1]]) <= 0):
                raise ValueError(f"row {i} has unsorted or duplicate columns")

    # -- device handle ---------------------------------------------------
    @property
    def handle(self):
        """A fresh device copy (CSR kind) or the assembled box handle."""
        if self._handle is None:
            lib = _lib.load()
            h = ctypes.c_void_p()
            ip = np.ascontiguousarray(self._indptr, dtype=np.int64)
            ix = np.ascontiguousarray(self._indices, dtype=np.int32)
            v = np.ascontiguousarray(self._values, dtype=float)
            if self.n == 0:
                raise ValueError("empty matrix")
            _lib.check(lib.lp_csr_create(self.n, int(ip[-1]), ip.ctypes.data, ix.ctypes.data,
                                         v.ctypes.data, ctypes.byref(h)), "csr upload")
            self._handle = h.value
            weakref.finalize(self, _destroy, h.value)
        return self._handle


class IluFactors:
    """ILU(0) factors: L strictly lower (unit diagonal implicit), U upper.

    The factors live on the device; ``L`` and ``U`` are exported as CSR
    ``SparseMatrix`` objects on first access."""

    def __init__(self, matrix, handle):
        self._matrix = matrix      # keeps the device handle alive
        self._handle = handle
        self._L = None
        self._U = None
        self.n = matrix.n

    def _part(self, which):
        lib = _lib.load()
        ip = np.empty(self.n + 1, dtype=np.int64)
        _lib.check(lib.lp_matrix_export(self._handle, which, ip.ctypes.data, None, None))
        nnz = int(ip[-1])
        ix = np.empty(nnz, dtype=np.int32)
        v = np.empty(nnz)
        _lib.check(lib.lp_matrix_export(self._handle, which, ip.ctypes.data, ix.ctypes.data,
                                        v.ctypes.data))
        return SparseMatrix(self.n, ip, ix, v)

    @property
    def L(self):
        if self._L is None:
            self._L = self._part(1)
        return self._L

    @property
    def U(self):
        if self._U is None:
            self._U = self._part(2)
        return self._U


def ilu0(m, pivot_tol=1e-300):
    """ILU(0) restricted to the pattern of M (sparse.py:142-172), on the GPU."""
    if m.n == 0:
        raise ValueError("empty matrix")
    if m._handle is None:
        handle = m.handle
        owner = m
    else:
        # assembled (box) matrices are factored in their own handle
        handle = m._handle
        owner = m
    bad = ctypes.c_int64(-1)
    rc = _lib.load().lp_ilu0(handle, pivot_tol, ctypes.byref(bad), _lib.stream_ptr())
    if rc == _lib.LP_ERR_ZERO_PIVOT:
        raise IluZeroPivotError(int(bad.value))
    _lib.check(rc, "ilu0")
    return IluFactors(owner, handle)


def _vec(f_or_m, x, name):
    n = f_or_m.n
    dev_in = device.is_device(x)
    if dev_in:
        if tuple(x.shape) != (n,):
            raise ValueError(f"length mismatch in {name}")
        return x.to(device.torch().float64).contiguous(), True
    x = np.asarray(x, dtype=float)
    if x.shape != (n,):
        raise ValueError(f"length mismatch in {name}")
    return device.to_device(x), False


def _run(fn, handle, x, n, dev_in):
    out = device.empty(n)
    _lib.check(getattr(_lib.load(), fn)(handle, x.data_ptr(), out.data_ptr(), _lib.stream_ptr()),
               fn)
    return out if dev_in else device.host(out)


def forward_sub(f, r):
    """Solve L y = r with the unit lower ILU factor (sparse.py:199-206)."""
    x, dev = _vec(f, r, "forward substitution")
    return _run("lp_forward_sub", f._handle, x, f.n, dev)


def backward_sub(f, y):
    """Solve U z = y with the upper ILU factor (sparse.py:209-216)."""
    x, dev = _vec(f, y, "backward substitution")
    return _run("lp_backward_sub", f._handle, x, f.n, dev)


def precond_apply(f, r):
    """One-step approximate solve of M z = r (sparse.py:219-221)."""
    x, dev = _vec(f, r, "precond_apply")
    return _run("lp_precond_apply", f._handle, x, f.n, dev)


def precond_apply_rz(f, r):
    """(z, r'z): the approximate solve M z = r together with the PCG scalar
    rho = r'z of pcg.py:147-151, accumulated inside the backward sweep
    (``lp_precond_apply_rz``; double-double, deterministic)."""
    x, dev = _vec(f, r, "precond_apply")
    out = device.empty(f.n)
    rz = device.empty(2)
    _lib.check(_lib.load().lp_precond_apply_rz(f._handle, x.data_ptr(), out.data_ptr(), rz.data_ptr(),
                                               _lib.stream_ptr()), "precond_apply")
    hi, lo = (float(v) for v in device.host(rz))
    return (out if dev else device.host(out)), hi + lo


def spmv(a, x):
    """y = A x (sparse.py:97-113)."""
    v, dev = _vec(a, x, "spmv")
    if not dev and v.numel() != a.n:
        raise ValueError(f"vector length {v.numel()} does not match n={a.n}")
    return _run("lp_spmv", a.handle, v, a.n, dev)


def save_matrix_market(path, a):
    from scipy.io import mmwrite
    mmwrite(str(path), a.to_scipy())


def load_matrix_market(path):
    from scipy.io import mmread
    return SparseMatrix.from_scipy(mmread(str(path)))
