"""Discrete Legendre transforms on the GPU (drop-in for transforms.py:27-375).

``TransformPlan(order)`` computes the Gauss rule on the host (bit-identical
to the reference) and hands the nodes and weights to the C ABI, which builds
the Vandermonde table and the Shen-basis tables on the device and keeps
them resident.  ``tensor_bdlt``/``tensor_fdlt`` run one parity-split DMMA
line-transform pass per axis.

The reference's "accelerated" mode (Toeplitz/Hankel + FFT) is not ported:
at the orders used here (P <= 2049) the dense contraction is both faster and
more accurate.  ``mode="accelerated"`` is accepted and runs the
dense path.
"""

from __future__ import annotations

import ctypes
import threading
import weakref

import numpy as np

from . import _lib, device
from .quadrature import gauss_rule

__all__ = ["TransformPlan", "bdlt", "fdlt", "tensor_bdlt", "tensor_fdlt",
           "transform_counter", "transform_count"]

_counts = threading.local()


def _bump():
    _counts.value = getattr(_counts, "value", 0) + 1


def transform_count():
    """Tensor transforms executed through this module on this thread."""
    return getattr(_counts, "value", 0)


class transform_counter:
    def __enter__(self):
        self._start = transform_count()
        return self

    def __exit__(self, *exc):
        self.count = transform_count() - self._start
        return False


def _destroy_plan(handle):
    try:
        _lib.load(init_device=False).lp_plan_destroy(handle)
    except Exception:
        pass


class TransformPlan:
    """Device-resident transform plan of order P (= N + 1)."""

    def __init__(self, order, mode="reference"):
        if mode not in ("reference", "accelerated"):
            raise ValueError(f"unknown transform mode {mode!r}")
        self.order = int(order)
        self.mode = mode
        self.rule = gauss_rule(self.order)
        self._fwd_scale = (2.0 * np.arange(self.order) + 1.0) / 2.0
        self._handle = None

    @property
    def handle(self):
        if self._handle is None:
            lib = _lib.load()
            h = ctypes.c_void_p()
            nodes = np.ascontiguousarray(self.rule.nodes)
            weights = np.ascontiguousarray(self.rule.weights)
            _lib.check(lib.lp_plan_create(self.order, nodes.ctypes.data, weights.ctypes.data,
                                          ctypes.byref(h)), "TransformPlan")
            self._handle = h.value
            weakref.finalize(self, _destroy_plan, h.value)
        return self._handle

    def table(self):
        """The P x P table V[k, n] = L_n(x_k) as built on the device."""
        out = np.empty((self.order, self.order))
        _lib.check(_lib.load().lp_plan_table(self.handle, out.ctypes.data))
        return out


def _tensor(fn_name, plan, a):
    dev_in = device.is_device(a)
    arr = a if dev_in else np.asarray(a, dtype=float)
    shape = tuple(arr.shape)
    if len(shape) not in (1, 2, 3):
        raise ValueError("tensor transforms support d = 1, 2, 3")
    if any(s != plan.order for s in shape):
        raise ValueError(f"all axes must have extent {plan.order}, got shape {shape}")
    _bump()
    src = device.to_device(arr)
    out = device.empty(src.numel())
    lib = _lib.load()
    _lib.check(getattr(lib, fn_name)(plan.handle, len(shape), src.data_ptr(), out.data_ptr(),
                                     _lib.stream_ptr()), fn_name)
    out = out.reshape(shape)
    return out if dev_in else device.host(out)


def tensor_bdlt(plan, coeffs):
    """Axis-wise backward transform f = V c of a P^d coefficient tensor."""
    return _tensor("lp_tensor_bdlt", plan, coeffs)


def tensor_fdlt(plan, values):
    """Axis-wise forward transform c_n = (2n+1)/2 sum_k w_k f_k L_n(x_k)."""
    return _tensor("lp_tensor_fdlt", plan, values)


def _vector(plan, x):
    x = np.asarray(x, dtype=float)
    if x.shape != (plan.order,):
        raise ValueError(f"expected a length-{plan.order} vector, got shape {x.shape}")
    return x


def bdlt(plan, coeffs):
    return tensor_bdlt(plan, _vector(plan, coeffs))


def fdlt(plan, values):
    return tensor_fdlt(plan, _vector(plan, values))
