"""Coefficient fields a(x), c(x), f(x) on (-1, 1)^d.

Mirrors the reference's ``CoefficientField`` contract
(``pkg/src/legpcg/coefficients.py:13-50``): a deterministic callable on
broadcastable coordinate arrays, an ``on_grid`` evaluation on a tensor grid
spanned by 1-D node arrays (``meshgrid(indexing="ij")``, axis 0 = x), and an
``is_zero`` flag so the reaction path can be skipped.

``LegendreSeriesField`` adds the seeded truncated-Legendre-series
coefficients of BASELINE configs 3 and 5 with a separable tensor-grid
evaluation (one small table per axis), so the P^3 = 513^3 grid of config 5
costs three small GEMMs instead of 12^3 passes over 1 GB.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np

__all__ = ["CoefficientField", "LegendreSeriesField", "zero_field",
           "constant_field", "PRESETS", "preset"]


@dataclass(frozen=True)
class CoefficientField:
    dim: int
    fn: Callable[..., np.ndarray]
    name: str = "<callable>"
    is_zero: bool = False

    def __call__(self, *coords):
        if len(coords) != self.dim:
            raise ValueError(f"field is {self.dim}-dimensional, "
                             f"got {len(coords)} coordinates")
        shape = np.broadcast_shapes(*(np.shape(c) for c in coords))
        vals = np.asarray(self.fn(*coords), dtype=float)
        return np.array(np.broadcast_to(vals, shape))

    def on_grid(self, axes):
        """Values on the tensor grid of the given 1-D node arrays (ij order)."""
        if len(axes) != self.dim:
            raise ValueError("one node array per dimension required")
        return self(*np.meshgrid(*axes, indexing="ij"))


def zero_field(dim):
    return CoefficientField(dim, lambda *c: 0.0, name="zero", is_zero=True)


def constant_field(dim, value, name=None):
    v = float(value)
    return CoefficientField(dim, lambda *c: v, name=name or f"const({value})",
                            is_zero=(v == 0.0))


def _legendre_rows(x, nmax):
    """rows[n] = L_n(x) for n = 0..nmax (three-term recurrence)."""
    x = np.asarray(x, dtype=float)
    rows = [np.ones_like(x)]
    if nmax >= 1:
        rows.append(x.copy())
    for k in range(1, nmax):
        rows.append(((2 * k + 1) * x * rows[k] - k * rows[k - 1]) / (k + 1))
    return rows


class LegendreSeriesField(CoefficientField):
    """offset + sum_{i,j,(k)} hat[i,j,(k)] L_i(x) L_j(y) (L_k(z))."""

    def __init__(self, hat, offset=0.0, name="series"):
        hat = np.asarray(hat, dtype=float)
        off = float(offset)

        def fn(*coords):
            acc = 0.0
            rows = [_legendre_rows(c, s - 1) for c, s in zip(coords, hat.shape)]
            for idx in np.ndindex(*hat.shape):
                term = hat[idx]
                for a, n in enumerate(idx):
                    term = term * rows[a][n]
                acc = acc + term
            return off + acc

        super().__init__(hat.ndim, fn, name=name, is_zero=False)
        object.__setattr__(self, "hat", hat)
        object.__setattr__(self, "offset", off)

    def on_grid(self, axes):
        if len(axes) != self.dim:
            raise ValueError("one node array per dimension required")
        out = self.hat
        for a, x in enumerate(axes):
            tab = np.stack(_legendre_rows(x, self.hat.shape[a] - 1), axis=1)
            out = np.moveaxis(np.tensordot(tab, out, axes=([1], [a])), 0, a)
        return self.offset + out


# --------------------------------------------------------------- presets
# The paper's examples (Tables 7-10) as named coefficient presets, the
# reference's `preset` / `PRESETS` contract (coefficients.py:53-127): a dict with
# dim, beta, alpha and axis_betas (per-axis 1-D diffusion factors) per name.

def _sq_norm(coords):
    return sum(np.asarray(c, dtype=float) ** 2 for c in coords)


def _quartic(*coords):            # (2|x|^2 + 1)^4
    return (2.0 * _sq_norm(coords) + 1.0) ** 4


def _exp_two_sum(*coords):        # e^{2(x + y + ...)}
    return np.exp(2.0 * sum(np.asarray(c, dtype=float) for c in coords))


def _cos_of_sum(*coords):         # cos(x + y + ...)
    return np.cos(sum(np.asarray(c, dtype=float) for c in coords))


_AXIS_FIELDS = {
    "exp2x": (lambda x: np.exp(2.0 * x), "e^{2x}"),
    "cosx": (np.cos, "cos(x)"),
    "expx": (np.exp, "e^x"),
    "cos_sin": (lambda x: np.cos(np.sin(x)), "cos(sin(x))"),
    "runge100": (lambda x: 1.0 / (1.0 + 100.0 * x * x), "1/(1+100x^2)"),
}


def _axis_field(key):
    fn, name = _AXIS_FIELDS[key]
    return CoefficientField(1, fn, name=name)


def _preset_table():
    t = {}

    def add(name, dim, beta=None, alpha=None, axis_betas=None):
        t[name] = {"dim": dim, "beta": beta, "alpha": alpha, "axis_betas": axis_betas}

    for d, tag in ((1, "1"), (2, "2"), (3, "3")):
        add(f"example{tag}a", d, beta=CoefficientField(d, _quartic, name="(2|x|^2+1)^4"),
            alpha=CoefficientField(d, _cos_of_sum, name="cos(sum x)"))
        add(f"example{tag}b", d, beta=CoefficientField(d, _exp_two_sum, name="e^{2 sum x}"),
            alpha=zero_field(d))
    add("example4a", 2, alpha=zero_field(2), axis_betas=(_axis_field("exp2x"), _axis_field("cosx")))
    add("example4b", 3, alpha=zero_field(3),
        axis_betas=(_axis_field("exp2x"), _axis_field("cosx"), _axis_field("cosx")))
    for key in ("expx", "cos_sin", "runge100"):     # 1-D rank-study fields
        add(key, 1, beta=_axis_field(key), alpha=_axis_field(key))
    return t


PRESETS = _preset_table()


def preset(name):
    """Named coefficient preset; KeyError for unknown names (coefficients.py:122-127)."""
    if name not in PRESETS:
        raise KeyError(f"unknown coefficient preset {name!r}")
    return PRESETS[name]
