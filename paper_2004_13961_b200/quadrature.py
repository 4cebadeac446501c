"""Host-side plan construction: Legendre-Gauss rules and Legendre tables.

These are setup computations (O(P^2) per plan) whose outputs seed the device
tables.  They restate ``legendre.py:86-145`` operation for operation so that
the nodes, weights and tables are bit-identical to the reference's -- which
keeps the GPU matvec about 1000x inside the 1e-12 parity bar at P = 2049
(SURVEY.md section 0.6).  The device rebuilds the same Vandermonde table from
these nodes with separately rounded operations (``operator.cu``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["GaussRule", "gauss_rule", "legendre_table", "phi_to_legendre",
           "dphi_to_legendre", "eval_legendre"]


@dataclass(frozen=True)
class GaussRule:
    order: int
    nodes: np.ndarray
    weights: np.ndarray


def _three_term(x, n):
    """(L_{n-1}(x), L_n(x)) by the upward recurrence, n >= 1."""
    lo, hi = np.ones_like(x), x.copy()
    k = 1
    while k < n:
        lo, hi = hi, ((2 * k + 1) * x * hi - k * lo) / (k + 1)
        k += 1
    return lo, hi


def _value_and_slope(n, x):
    prev, cur = _three_term(x, n)
    return cur, n * (prev - x * cur) / (1.0 - x * x)


_RULES = {}


def gauss_rule(order, tol=1e-15, max_iter=100):
    """Nodes (increasing) and weights of the order-P Legendre-Gauss rule.

    Newton iteration from cos(pi (4k+3)/(4P+2)) with
    (1 - x^2) L_P' = P (L_{P-1} - x L_P), one polishing step, then exact
    antisymmetrisation of the nodes and symmetrisation of the weights.
    Rules are memoised (read-only arrays): every solve's setup asks for the
    same few orders."""
    key = (int(order), float(tol), int(max_iter))
    rule = _RULES.get(key)
    if rule is None:
        rule = _gauss_rule(*key)
        rule.nodes.flags.writeable = False
        rule.weights.flags.writeable = False
        _RULES[key] = rule
    return rule


def _gauss_rule(order, tol, max_iter):
    P = int(order)
    if P < 1:
        raise ValueError("order must be >= 1")
    if P == 1:
        return GaussRule(1, np.zeros(1), np.full(1, 2.0))
    x = np.cos(np.pi * (4 * np.arange(P) + 3) / (4 * P + 2))
    converged = False
    for _ in range(max_iter):
        val, slope = _value_and_slope(P, x)
        step = val / slope
        x -= step
        if np.max(np.abs(step)) < tol:
            converged = True
            break
    if not converged:
        raise RuntimeError(f"Gauss-Newton iteration for order {P} did not converge")
    val, slope = _value_and_slope(P, x)
    x -= val / slope
    x = np.flip(x).copy()
    x = 0.5 * (x - np.flip(x))
    _, slope = _value_and_slope(P, x)
    w = 2.0 / ((1.0 - x * x) * slope * slope)
    w = 0.5 * (w + np.flip(w))
    return GaussRule(P, x, w)


def legendre_table(x, nmax):
    """T[j, n] = L_n(x_j), n = 0..nmax (host copy, same recurrence)."""
    x = np.asarray(x, dtype=float)
    cols = [np.ones_like(x)]
    if nmax >= 1:
        cols.append(x.copy())
    for k in range(1, nmax):
        cols.append(((2 * k + 1) * x * cols[k] - k * cols[k - 1]) / (k + 1))
    return np.stack(cols, axis=1) if cols else np.empty((x.size, 0))


def eval_legendre(n, x):
    x = np.asarray(x, dtype=float)
    if n == 0:
        out = np.ones_like(x)
    else:
        out = _three_term(x, n)[1]
    return out if out.ndim else float(out)


def phi_to_legendre(u, axis=-1):
    """Shen coefficients -> Legendre coefficients: out_k = u_k - u_{k-2}."""
    u = np.moveaxis(np.asarray(u, dtype=float), axis, -1)
    out = np.zeros(u.shape[:-1] + (u.shape[-1] + 2,))
    out[..., :-2] = u
    out[..., 2:] -= u
    return np.moveaxis(out, -1, axis)


def dphi_to_legendre(u, axis=-1):
    """Legendre coefficients of the derivative: out_{k+1} = -(2k+3) u_k."""
    u = np.moveaxis(np.asarray(u, dtype=float), axis, -1)
    k = u.shape[-1]
    out = np.zeros(u.shape[:-1] + (k + 2,))
    out[..., 1:k + 1] = -(2.0 * np.arange(k) + 3.0) * u
    return np.moveaxis(out, -1, axis)
