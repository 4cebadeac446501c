"""Matrix-free Galerkin operator on the GPU (drop-in for operator.py:21-222).

``apply_A`` / ``apply_B`` / ``apply_system`` keep the reference signatures and
return ``SpectralCoeffs``; the work runs in ``lp_apply`` (csrc/operator.cu), a
sum-factorised evaluation of exactly the pipeline of operator.py:161-187
(phi->Legendre conversion, BDLT, pointwise coefficient product, FDLT,
closed-form contraction), 2d parity-split DMMA line-transform passes per call.

Inputs may be numpy arrays (copied to and from the device, the reference's
by-value semantics) or CUDA tensors (kept resident; same K^d shape, axis 0 = x).
"""

from __future__ import annotations

import ctypes
import weakref
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib, device
from .coefficients import CoefficientField, LegendreSeriesField
from .transforms import TransformPlan, tensor_fdlt

__all__ = ["SpectralCoeffs", "ProblemSpec", "apply_A", "apply_B", "apply_system",
           "assemble_rhs"]


@dataclass
class SpectralCoeffs:
    """Boundary-adapted (Shen) coefficient tensor of shape K^d, axis 0 = x."""

    data: object

    def __post_init__(self):
        if device.is_device(self.data):
            t = device.torch()
            self.data = self.data.to(t.float64)
            shape = tuple(self.data.shape)
            finite = bool(t.isfinite(self.data).all())
        else:
            self.data = np.asarray(self.data, dtype=float)
            shape = self.data.shape
            finite = bool(np.all(np.isfinite(self.data)))
        k = shape[0] if len(shape) else 0
        if len(shape) not in (1, 2, 3) or any(s != k for s in shape) or k < 1:
            raise ValueError(f"coefficient tensor must be K^d with d in 1..3, got shape {shape}")
        if not finite:
            raise ValueError("coefficient tensor contains non-finite entries")

    @property
    def dim(self):
        return len(self.data.shape)

    @property
    def n_modes(self):
        return self.data.shape[0]


def _destroy_op(handle):
    try:
        _lib.load(init_device=False).lp_operator_destroy(handle)
    except Exception:
        pass


@dataclass
class ProblemSpec:
    """Dimension, cutoff N and coefficient fields (operator.py:59-120)."""

    dim: int
    N: int
    beta: Optional[CoefficientField] = None
    alpha: Optional[CoefficientField] = None
    rhs: Optional[CoefficientField] = None
    axis_betas: Optional[Sequence[CoefficientField]] = None
    _grid_cache: dict = field(default_factory=dict, repr=False, compare=False)
    _op_cache: dict = field(default_factory=dict, repr=False, compare=False)

    def __post_init__(self):
        if self.N < 3:
            raise ValueError("polynomial cutoff N must be >= 3")
        if self.dim not in (1, 2, 3):
            raise ValueError("dim must be 1, 2 or 3")
        if (self.beta is None) == (self.axis_betas is None):
            raise ValueError("exactly one of beta / axis_betas is required")
        if self.axis_betas is not None and len(self.axis_betas) != self.dim:
            raise ValueError("axis_betas must supply one 1-D field per axis")

    @property
    def n_modes(self):
        return self.N - 1

    @property
    def has_reaction(self):
        return self.alpha is not None and not self.alpha.is_zero

    def _check_plan(self, plan):
        if plan.order != self.N + 1:
            raise ValueError(f"plan order {plan.order} does not match N + 1 = {self.N + 1}")

    def grid_values(self, plan, role, positivity_floor=None):
        """Coefficient values on the tensor Gauss grid (ij order, axis 0 = x)."""
        key = (role, plan.order)
        if key not in self._grid_cache:
            if isinstance(role, tuple):
                i = role[1]
                vals = self.axis_betas[i](plan.rule.nodes)
                shape = [1] * self.dim
                shape[i] = plan.order
                self._grid_cache[key] = vals.reshape(shape)
            else:
                fld = {"beta": self.beta, "alpha": self.alpha, "rhs": self.rhs}[role]
                if fld is None:
                    raise ValueError(f"problem spec has no {role} field")
                self._grid_cache[key] = fld.on_grid([plan.rule.nodes] * self.dim)
        vals = self._grid_cache[key]
        if positivity_floor is not None and np.min(vals) <= positivity_floor:
            raise ValueError(f"diffusion coefficient is not positive on the grid "
                             f"(min {np.min(vals):.3e})")
        return vals

    def device_operator(self, plan):
        """lp_operator handle for (spec, plan): weighted grids resident on the GPU."""
        self._check_plan(plan)
        key = plan.order
        if key not in self._op_cache:
            lib = _lib.load()
            d = self.dim
            h = ctypes.c_void_p()
            keep = []
            if self.axis_betas is not None:
                arrs = [np.ascontiguousarray(f(plan.rule.nodes), dtype=float)
                        for f in self.axis_betas]
                keep += arrs
                ptrs = (ctypes.c_void_p * d)(*[a.ctypes.data for a in arrs])
                beta_ptr, nab = None, d
            else:
                g = _series_grid_on_device(self.beta, plan, d)
                if g is None:
                    # x-fastest device order = transpose of the ij-indexed grid
                    g = np.ascontiguousarray(self.grid_values(plan, "beta").T)
                    beta_ptr = g.ctypes.data
                else:
                    beta_ptr = g.data_ptr()
                keep.append(g)
                nab, ptrs = 0, None
            alpha_ptr = None
            if self.has_reaction:
                ga = _series_grid_on_device(self.alpha, plan, d)
                if ga is None:
                    ga = np.ascontiguousarray(
                        np.broadcast_to(self.grid_values(plan, "alpha"), (plan.order,) * d).T)
                    alpha_ptr = ga.ctypes.data
                else:
                    alpha_ptr = ga.data_ptr()
                keep.append(ga)
            _lib.check(lib.lp_operator_create(plan.handle, d, beta_ptr, nab, ptrs, alpha_ptr,
                                              ctypes.byref(h)), "operator")
            self._op_cache[key] = (h.value, plan)
            weakref.finalize(self, _destroy_op, h.value)
            if any(not isinstance(k, np.ndarray) for k in keep):
                # device-built grids were copied into the operator: hand their
                # memory back (the preconditioner of cfg 5 needs ~140 GB next)
                del keep
                device.torch().cuda.empty_cache()
        return self._op_cache[key][0]


def _series_grid_on_device(fld, plan, d):
    """Values of a truncated Legendre series field on the P^d Gauss grid, built on
    the GPU: the tensor BDLT of the zero-padded hat, with the
    offset folded into the L_0...L_0 coefficient.  This is the grid_values of
    operator.py:95-120 for these fields (the series is exact at the nodes), without
    the host P^d evaluation and upload (cfg 5: two 1.08 GB grids).  None for other
    fields, which are user callables evaluated on the host."""
    if not isinstance(fld, LegendreSeriesField) or fld.dim != d:
        return None
    P = plan.order
    if any(s > P for s in fld.hat.shape):
        return None
    pad = np.zeros((P,) * d)
    pad[tuple(slice(0, s) for s in fld.hat.shape)] = fld.hat
    pad[(0,) * d] += fld.offset
    src = device.to_device(pad.flatten(order="F"))      # x fastest
    out = device.empty(P ** d)
    _lib.check(_lib.load().lp_tensor_bdlt(plan.handle, d, src.data_ptr(), out.data_ptr(),
                                          _lib.stream_ptr()), "series grid")
    device.torch().cuda.current_stream().synchronize()
    return out


def _check_input(spec, plan, u):
    spec._check_plan(plan)
    if u.dim != spec.dim or u.n_modes != spec.n_modes:
        raise ValueError(f"coefficient tensor shape {tuple(u.data.shape)} does not match "
                         f"dim={spec.dim}, K={spec.n_modes}")


def apply_flat(spec, plan, which, u_flat):
    """Device x-fastest vector in, device vector out (no layout changes)."""
    out = device.empty(u_flat.numel())
    _lib.check(_lib.load().lp_apply(spec.device_operator(plan), which, u_flat.data_ptr(),
                                    out.data_ptr(), _lib.stream_ptr()), "apply")
    return out


def apply_flat_dot(spec, plan, which, u_flat):
    """(out, u'out): the matvec with the PCG curvature p'w (pcg.py:156-157)
    accumulated inside its last pass (``lp_apply_dot``; double-double,
    deterministic).  Device x-fastest vector in, device vector and float out."""
    out = device.empty(u_flat.numel())
    uw = device.empty(2)
    _lib.check(_lib.load().lp_apply_dot(spec.device_operator(plan), which, u_flat.data_ptr(),
                                        out.data_ptr(), uw.data_ptr(), _lib.stream_ptr()), "apply")
    hi, lo = (float(v) for v in device.host(uw))
    return out, hi + lo


def _apply(spec, plan, u, which):
    _check_input(spec, plan, u)
    dev_in = device.is_device(u.data)
    flat = device.to_device(device.fortran_flat(u.data))
    out = apply_flat(spec, plan, which, flat)
    if not dev_in:
        out = device.host(out)
    return SpectralCoeffs(device.from_fortran_flat(out, spec.n_modes, spec.dim))


def apply_A(spec, plan, u):
    """Diffusion matrix action A u without forming A (operator.py:190-192)."""
    return _apply(spec, plan, u, 1)


def apply_B(spec, plan, u):
    """Reaction matrix action B u (operator.py:195-201)."""
    if not spec.has_reaction:
        _check_input(spec, plan, u)
        z = u.data * 0.0
        return SpectralCoeffs(z)
    return _apply(spec, plan, u, 2)


def apply_system(spec, plan, u):
    """(A + B) u; the reaction path is skipped when alpha is zero (operator.py:204-210)."""
    return _apply(spec, plan, u, 3)


def mass_contract(v, axis):
    """out_k = 2 v_k/(2k+1) - 2 v_{k+2}/(2k+5) along ``axis`` (P -> K)."""
    m = np.moveaxis(np.asarray(v, dtype=float), axis, -1)
    k = m.shape[-1] - 2
    ks = np.arange(k, dtype=float)
    out = (2.0 / (2 * ks + 1)) * m[..., :k] - (2.0 / (2 * ks + 5)) * m[..., 2:]
    return np.moveaxis(out, -1, axis)


def mass_contract_device(fhat_flat, dim, P):
    """All-axes mass contraction of a device P^d Legendre coefficient vector
    (x fastest) on the GPU: K^d device vector (``lp_mass_contract``)."""
    out = device.empty((P - 2) ** dim)
    _lib.check(_lib.load().lp_mass_contract(dim, P, fhat_flat.data_ptr(), out.data_ptr(),
                                            _lib.stream_ptr()), "mass contraction")
    return out


def assemble_rhs(spec, plan):
    """Load vector F_k = (I_N f, phi_k) (operator.py:213-222): GPU FDLT of the
    sampled f, then the closed-form mass contraction per axis, also on the GPU
    (bit-identical to the reference's numpy expression)."""
    spec._check_plan(plan)
    if spec.rhs is None:
        raise ValueError("problem spec has no right-hand-side field")
    d, P = spec.dim, plan.order
    vals = device.to_device(device.fortran_flat(np.broadcast_to(
        spec.grid_values(plan, "rhs"), (P,) * d)))
    fh = device.empty(P ** d)
    lib = _lib.load()
    _lib.check(lib.lp_tensor_fdlt(plan.handle, d, vals.data_ptr(), fh.data_ptr(), _lib.stream_ptr()),
               "assemble_rhs")
    out = mass_contract_device(fh, d, P)
    return SpectralCoeffs(device.from_fortran_flat(device.host(out), spec.n_modes, d))
