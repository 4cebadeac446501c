"""Seeded synthetic workloads for the five BASELINE.json configurations.

The reference ships no dataset; BASELINE.json fixes the shapes and value
distributions and SURVEY.md section 8(d) the recipe.  Every input is built once on the
host from fixed seeds so that the GPU path, the CPU oracle and the reference
see identical arrays:

* cfg 1 -- 1-D N=128, a = 2 + sin(pi x), c = 1 + x^2, f from the manufactured
  solution u = (1 - x^2) e^x sin(pi x); F = assemble_rhs(f); T = 8, rtol 1e-12.
* cfg 2 -- 2-D N=256, a = 1 + 0.5 cos(pi x) cos(pi y) + 0.25 x y,
  c = exp(x + y); f_hat_ij = g_ij / ((i+1)(j+1)), g iid N(0,1); T = 10.
* cfg 3 -- 2-D N=2048, a = 3 + 16x16 series, c = 1 + 16x16 series, series
  coefficients U(-1,1) * 2^-(i+j); T = 12.
* cfg 4 -- 3-D N=128, a = 2 + sin sin sin + 0.3 |x|^2, c = 1; T = 8.
* cfg 5 -- 3-D N=512, a = 4 + 12^3 series, c = 1 + 12^3 series; T = 8.

For the f_hat configs the load vector is F = per-axis mass contraction of the
P^d Legendre series f_hat (``operator.py:131-144`` applied to the series), i.e.
``assemble_rhs`` of that series up to rounding.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from .coefficients import (CoefficientField, LegendreSeriesField,
                           constant_field)

SEED_RHS = 2004
SEED_COEF = 13961


@dataclass
class Workload:
    name: str
    dim: int
    N: int
    T: int
    rtol: float
    beta: CoefficientField
    alpha: Optional[CoefficientField]
    rhs_field: Optional[CoefficientField] = None   # cfg 1: f(x) sampled at Gauss nodes
    fhat: Optional[np.ndarray] = None               # other cfgs: P^d Legendre series of f

    @property
    def K(self):
        return self.N - 1

    @property
    def P(self):
        return self.N + 1

    @property
    def dofs(self):
        return self.K ** self.dim


def mass_contract_series(fhat):
    """F_k = 2 f_k/(2k+1) - 2 f_{k+2}/(2k+5) along every axis (P^d -> K^d)."""
    h = np.asarray(fhat, dtype=float)
    for ax in range(h.ndim):
        m = np.moveaxis(h, ax, 0)
        k = m.shape[0] - 2
        ks = np.arange(k, dtype=float).reshape((k,) + (1,) * (m.ndim - 1))
        h = np.moveaxis((2.0 / (2 * ks + 1)) * m[:k] - (2.0 / (2 * ks + 5)) * m[2:], 0, ax)
    return h


def rhs_on_device(fhat):
    """The same load vector built on the GPU: the P^d series coefficients are
    uploaded once and contracted there (``lp_mass_contract``, bit-identical to
    ``mass_contract_series``); returns the x-fastest device vector of K^d."""
    from . import device
    from .operator import mass_contract_device
    h = np.asarray(fhat, dtype=float)
    return mass_contract_device(device.to_device(h.flatten(order="F")), h.ndim, h.shape[0])


def seeded_fhat(dim, P, seed=SEED_RHS):
    g = np.random.default_rng(seed).standard_normal((P,) * dim)
    scale = np.ones(())
    for ax in range(dim):
        shp = [1] * dim
        shp[ax] = P
        scale = scale * (1.0 / (np.arange(P) + 1.0)).reshape(shp)
    return g * scale


def seeded_series(dim, nterms, offset, seed, name):
    rng = np.random.default_rng(seed)
    hat = rng.uniform(-1.0, 1.0, (nterms,) * dim)
    idx = np.indices((nterms,) * dim).sum(axis=0)
    return LegendreSeriesField(hat * 2.0 ** (-idx.astype(float)), offset, name)


def _manufactured_1d():
    pi = np.pi

    def f(x):
        e, s, c = np.exp(x), np.sin(pi * x), np.cos(pi * x)
        g, dg, ddg = 1.0 - x * x, -2.0 * x, -2.0
        h = e * s
        dh = e * (s + pi * c)
        ddh = e * ((1.0 - pi * pi) * s + 2.0 * pi * c)
        u = g * h
        du = dg * h + g * dh
        ddu = ddg * h + 2.0 * dg * dh + g * ddh
        a, da = 2.0 + s, pi * c
        return -(da * du + a * ddu) + (1.0 + x * x) * u

    def u_exact(x):
        return (1.0 - x * x) * np.exp(x) * np.sin(pi * x)

    return CoefficientField(1, f, name="f_manufactured"), u_exact


def cfg1(N=128):
    f, _ = _manufactured_1d()
    return Workload("cfg1", 1, N, 8, 1e-12,
                    beta=CoefficientField(1, lambda x: 2.0 + np.sin(np.pi * x), "2+sin(pi x)"),
                    alpha=CoefficientField(1, lambda x: 1.0 + x * x, "1+x^2"),
                    rhs_field=f)


def cfg2(N=256, T=10):
    beta = CoefficientField(
        2, lambda x, y: 1.0 + 0.5 * np.cos(np.pi * x) * np.cos(np.pi * y) + 0.25 * x * y,
        "1+0.5cos(pi x)cos(pi y)+0.25xy")
    alpha = CoefficientField(2, lambda x, y: np.exp(x + y), "exp(x+y)")
    return Workload("cfg2", 2, N, T, 1e-10, beta, alpha, fhat=seeded_fhat(2, N + 1))


def cfg3(N=2048, T=12):
    beta = seeded_series(2, 16, 3.0, SEED_COEF, "3+series16")
    alpha = seeded_series(2, 16, 1.0, SEED_COEF + 1, "1+series16")
    return Workload("cfg3", 2, N, T, 1e-10, beta, alpha, fhat=seeded_fhat(2, N + 1))


def cfg4(N=128, T=8):
    beta = CoefficientField(
        3, lambda x, y, z: 2.0 + np.sin(np.pi * x) * np.sin(np.pi * y) * np.sin(np.pi * z)
        + 0.3 * (x * x + y * y + z * z), "2+sinsinsin+0.3|x|^2")
    return Workload("cfg4", 3, N, T, 1e-10, beta, constant_field(3, 1.0),
                    fhat=seeded_fhat(3, N + 1))


def cfg5(N=512, T=8):
    beta = seeded_series(3, 12, 4.0, SEED_COEF + 2, "4+series12")
    alpha = seeded_series(3, 12, 1.0, SEED_COEF + 3, "1+series12")
    return Workload("cfg5", 3, N, T, 1e-10, beta, alpha, fhat=seeded_fhat(3, N + 1))


CONFIGS = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4, "cfg5": cfg5}


def manufactured_solution_1d():
    return _manufactured_1d()[1]
