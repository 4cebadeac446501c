"""CPU-only tests: the C ABI library loads and exports every declared symbol,
and the host-side setup code of the package matches the reference."""

import ctypes
import os
import re

import numpy as np
import pytest

from oracle import legpcg_port as orc
from paper_2004_13961_b200 import _lib, quadrature, precond, workloads as wl
from paper_2004_13961_b200.operator import ProblemSpec, SpectralCoeffs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "legpcg_b200.h")).read()
    return sorted(set(re.findall(r"\b(lp_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built")
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 20
    for name in syms:
        assert hasattr(lib, name), name
    assert set(syms) == set(_lib.EXPORTED)


def test_library_reports_no_device_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available() or not os.path.exists(_lib.LIB_PATH):
        pytest.skip("GPU present or library missing")
    lib = _lib.load(init_device=False)
    assert lib.lp_init(0) == _lib.LP_ERR_NODEVICE
    assert b"device" in lib.lp_last_error()


@pytest.mark.parametrize("P", [1, 2, 3, 5, 17, 33, 64, 129, 257, 513, 2049])
def test_host_gauss_rule_bitwise(golden, P):
    g = golden("quadrature")
    r = quadrature.gauss_rule(P)
    np.testing.assert_array_equal(r.nodes, g[f"gauss{P}_nodes"])
    np.testing.assert_array_equal(r.weights, g[f"gauss{P}_weights"])


def test_host_legendre_table_bitwise(golden):
    g = golden("quadrature")
    np.testing.assert_array_equal(quadrature.legendre_table(g["gauss33_nodes"], 32), g["table33"])


def test_phi_maps_known_answers():
    # reference tests/test_legendre.py:152-168
    np.testing.assert_array_equal(quadrature.phi_to_legendre(np.array([1.0])), [1.0, 0.0, -1.0])
    np.testing.assert_array_equal(quadrature.dphi_to_legendre(np.array([1.0])), [0.0, -3.0, 0.0])


@pytest.mark.parametrize("name,t", [("cfg1", 8), ("cfg2", 10), ("cfg3", 12), ("cfg4", 8)])
def test_expand_coefficient_bitwise_vs_oracle(name, t):
    w = wl.CONFIGS[name]()
    a = precond.expand_coefficient(w.beta, t, w.dim).hat
    b = orc.expand_coefficient(w.beta, t, w.dim)
    np.testing.assert_array_equal(a, b)


def test_building_blocks_insufficient_quadrature():
    with pytest.raises(ValueError, match="quadrature order"):
        precond.building_blocks_1d(4, 20, quadrature.gauss_rule(12))


def test_predicted_bandwidth_table():
    pb = precond.predicted_bandwidth
    assert pb(0, "even", "diffusion") == 1 and pb(0, "even", "reaction") == 5
    assert (pb(2, "odd", "diffusion"), pb(3, "odd", "diffusion")) == (3, 7)
    assert (pb(2, "even", "diffusion"), pb(3, "even", "diffusion")) == (5, 5)
    assert (pb(2, "odd", "reaction"), pb(3, "odd", "reaction")) == (7, 11)
    assert (pb(2, "even", "reaction"), pb(3, "even", "reaction")) == (9, 9)
    with pytest.raises(ValueError):
        pb(2, "mixed", "diffusion")


def test_spec_and_coeff_validation():
    with pytest.raises(ValueError):
        ProblemSpec(dim=2, N=2, beta=wl.constant_field(2, 1.0))
    with pytest.raises(ValueError):
        ProblemSpec(dim=4, N=8, beta=wl.constant_field(2, 1.0))
    with pytest.raises(ValueError):
        ProblemSpec(dim=2, N=8)
    with pytest.raises(ValueError):
        SpectralCoeffs(np.ones((3, 4)))
    with pytest.raises(ValueError):
        SpectralCoeffs(np.array([1.0, np.nan]))


def test_series_field_separable_grid_matches_pointwise():
    f = wl.seeded_series(2, 16, 3.0, 5, "s")
    x = quadrature.gauss_rule(40).nodes
    np.testing.assert_allclose(f.on_grid([x, x]), f(*np.meshgrid(x, x, indexing="ij")),
                               rtol=1e-13, atol=1e-13)


def test_workload_coefficients_positive():
    # BASELINE series coefficients can in principle be <= 0; the seeds used are not
    for name in ("cfg3", "cfg5"):
        w = wl.CONFIGS[name]()
        x = quadrature.gauss_rule(65).nodes
        assert np.min(w.beta.on_grid([x] * w.dim)) > 0
