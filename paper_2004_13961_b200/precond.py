"""Truncated-coefficient preconditioner M (drop-in for precond.py:26-318).

``expand_coefficient`` truncates each coefficient to a degree-t Legendre series
on a 32-point grid (host: the fields are Python callables, 32^d samples).
``building_blocks_1d`` -- the diagonals of the exact-quadrature 1-D blocks
S^(t), M^(t) -- runs on the GPU (``lp_blocks_1d``), and so does the K^d-sized
work: the hat-weighted sum of Kronecker products, the symmetrisation and the
pattern/compression
(``lp_box_assemble``) straight into the implicit-offset layout the ILU(0)
kernels consume; no CSR is built unless the caller asks for it.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .quadrature import GaussRule, gauss_rule, legendre_table
from .sparse import SparseMatrix

__all__ = ["TruncatedCoefficient", "BandedBlock", "expand_coefficient",
           "building_blocks_1d", "assemble_M", "predicted_bandwidth"]

@dataclass(frozen=True)
class TruncatedCoefficient:
    dim: int
    t: int
    hat: np.ndarray

    def __post_init__(self):
        if self.hat.shape != (self.t + 1,) * self.dim:
            raise ValueError(f"hat tensor shape {self.hat.shape} does not match "
                             f"(t+1)^d = {(self.t + 1,) * self.dim}")

    def evaluate(self, axes):
        out = self.hat
        for a, x in enumerate(axes):
            tab = legendre_table(np.asarray(x, dtype=float), self.t)
            out = np.moveaxis(np.tensordot(tab, out, axes=([1], [a])), 0, a)
        return out


def _host_fdlt(order, values):
    """Axis-wise FDLT on the small expansion grid (transforms.py:319-325)."""
    rule = gauss_rule(order)
    tab = legendre_table(rule.nodes, order - 1)
    scale = (2.0 * np.arange(order) + 1.0) / 2.0
    a = np.asarray(values, dtype=float)
    for ax in range(a.ndim):
        m = np.moveaxis(a, ax, 0)
        shp = m.shape
        flat = np.ascontiguousarray(m.reshape(shp[0], -1))
        res = scale[:, None] * (tab.T @ (rule.weights[:, None] * flat))
        a = np.moveaxis(res.reshape(shp), 0, ax)
    return a, rule


def expand_coefficient(field, t, dim):
    """Degree-t truncation sampled on max(2(t+1), 32) Gauss points (precond.py:75-87)."""
    if t < 0:
        raise ValueError("cutoff t must be nonnegative")
    p = max(2 * (t + 1), 32)
    rule = gauss_rule(p)
    hat, _ = _host_fdlt(p, field.on_grid([rule.nodes] * dim))
    return TruncatedCoefficient(dim, t, hat[(slice(0, t + 1),) * dim].copy())


@dataclass(frozen=True)
class BandedBlock:
    kind: str
    t: int
    size: int
    diags: dict

    def to_dense(self):
        a = np.zeros((self.size, self.size))
        for o, d in self.diags.items():
            rows = np.arange(max(0, -o), self.size - max(0, o))
            a[rows, rows + o] = d[rows]
        return a


def _offsets(kind, t):
    reach = t if kind == "stiff" else t + 2
    return [o for o in range(-reach, reach + 1) if (o - t) % 2 == 0]


_BLOCKS = {}


def _block_stack(T, K, rule):
    """blocks[kind][t][o + R][i] = entry (i, i+o) of S^(t) (kind 0) / M^(t)
    (kind 1), R = T + 2: the exact-quadrature diagonals, computed on the GPU
    (``lp_blocks_1d``) in the reference's operation order (precond.py:118-161:
    nodes in order, a partial sum per chunk of 512 nodes), so they are
    bit-identical to the reference's.  Memoised per (T, K, rule)."""
    key = (int(T), int(K), rule.nodes.tobytes(), rule.weights.tobytes())
    hit = _BLOCKS.get(key)
    if hit is None:
        R = T + 2
        hit = np.zeros((2, T + 1, 2 * R + 1, K))
        nodes = np.ascontiguousarray(rule.nodes, dtype=float)
        weights = np.ascontiguousarray(rule.weights, dtype=float)
        _lib.check(_lib.load().lp_blocks_1d(int(T), int(K), int(rule.order), nodes.ctypes.data,
                                            weights.ctypes.data, hit.ctypes.data), "building_blocks_1d")
        hit.flags.writeable = False
        _BLOCKS[key] = hit
    return hit


def building_blocks_1d(T, K, plan):
    """Exact-quadrature diagonals of S^(t) = (L_t phi', phi') and
    M^(t) = (L_t phi, phi), t = 0..T (precond.py:118-161), as read-only
    ``BandedBlock`` views of the GPU-built stack."""
    if T < 0 or K < 1:
        raise ValueError("need T >= 0 and K >= 1")
    rule = plan if isinstance(plan, GaussRule) else plan.rule
    needed = K + T // 2 + 2
    if rule.order < needed:
        raise ValueError(f"quadrature order {rule.order} is insufficient for exact "
                         f"blocks with T={T}, K={K}: need at least {needed}")
    stack = _block_stack(int(T), int(K), rule)
    R = T + 2
    out = []
    for kind, name in enumerate(("stiff", "mass")):
        out.append([BandedBlock(name, t, K, {o: stack[kind, t, o + R] for o in _offsets(name, t)})
                    for t in range(T + 1)])
    return out[0], out[1]


def _groups(spec, t1, t2):
    """(hat, stiff axis or None) terms (precond.py:175-197), cached on the spec
    (its coefficient fields are fixed)."""
    key = ("groups", tuple(t1) if isinstance(t1, (tuple, list)) else t1, t2)
    hit = spec._op_cache.get(key)
    if hit is None:
        hit = _groups_uncached(spec, t1, t2)
        spec._op_cache[key] = hit
    return hit


def _groups_uncached(spec, t1, t2):
    d = spec.dim
    out = []
    if spec.axis_betas is not None:
        cuts = t1 if isinstance(t1, (tuple, list)) else (t1,) * d
        if len(cuts) != d:
            raise ValueError("one diffusion cutoff per axis required")
        for i in range(d):
            h1 = expand_coefficient(spec.axis_betas[i], cuts[i], 1).hat
            shape = [1] * d
            shape[i] = cuts[i] + 1
            out.append((h1.reshape(shape), i))
    else:
        hat = expand_coefficient(spec.beta, int(t1), d).hat
        out += [(hat, i) for i in range(d)]
    if spec.alpha is not None and not spec.alpha.is_zero:
        out.append((expand_coefficient(spec.alpha, int(t2), d).hat, None))
    return out


def assemble_M(spec, t1, t2, plan=None):
    """Assemble the preconditioner on the GPU; returns a device-resident
    ``SparseMatrix`` (x index fastest, symmetric by construction)."""
    d, K = spec.dim, spec.n_modes
    if K < 1:
        raise ValueError("empty preconditioner: K = 0")
    groups = _groups(spec, t1, t2)
    tmax = max(h.shape[a] for h, _ in groups for a in range(d)) - 1
    rule = gauss_rule(K + tmax // 2 + 2)
    blocks = _block_stack(tmax, K, rule)
    lens = np.array([h.shape for h, _ in groups], dtype=np.int32).reshape(-1)
    stiff = np.array([-1 if s is None else s for _, s in groups], dtype=np.int32)
    hats = [np.ascontiguousarray(h, dtype=float) for h, _ in groups]
    hat_ptrs = (ctypes.c_void_p * len(hats))(*[h.ctypes.data for h in hats])
    h = ctypes.c_void_p()
    _lib.check(_lib.load().lp_box_assemble(d, K, len(groups), lens.ctypes.data,
                                           stiff.ctypes.data, hat_ptrs, tmax,
                                           blocks.ctypes.data, ctypes.byref(h)), "assemble_M")
    return SparseMatrix(K ** d, _handle=h.value)


def predicted_bandwidth(t, parity, which):
    """Proposition 4.1 band widths (precond.py:300-318)."""
    if parity not in ("even", "odd"):
        raise ValueError("parity must be 'even' or 'odd'")
    even_t = t % 2 == 0
    if which == "diffusion":
        wide = (parity == "even") == even_t
        return 2 * t + 1 if wide else 2 * t - 1
    if which == "reaction":
        wide = (parity == "even") == even_t
        return 2 * t + 5 if wide else 2 * t + 3
    raise ValueError("which must be 'diffusion' or 'reaction'")
