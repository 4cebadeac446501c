"""Paper-table benchmark registry and run_benchmark (pcg.py:182-271) on the GPU path."""

import numpy as np
import pytest

from paper_2004_13961_b200 import BENCHMARKS, PRESETS, benchmark_rhs, make_problem, preset


def test_presets_closed_forms():
    rng = np.random.default_rng(4)
    x, y, z = rng.uniform(-1, 1, (3, 50))
    p = preset("example3a")
    np.testing.assert_allclose(p["beta"](x, y, z), (2 * (x * x + y * y + z * z) + 1) ** 4, rtol=1e-15)
    np.testing.assert_allclose(p["alpha"](x, y, z), np.cos(x + y + z), rtol=1e-15)
    p = preset("example2b")
    np.testing.assert_allclose(p["beta"](x, y), np.exp(2 * (x + y)), rtol=1e-15)
    assert p["alpha"].is_zero
    p = preset("example4b")
    assert p["beta"] is None and len(p["axis_betas"]) == 3
    np.testing.assert_allclose(p["axis_betas"][0](x), np.exp(2 * x), rtol=1e-15)
    np.testing.assert_allclose(p["axis_betas"][2](x), np.cos(x), rtol=1e-15)
    np.testing.assert_allclose(preset("runge100")["beta"](x), 1 / (1 + 100 * x * x), rtol=1e-15)
    with pytest.raises(KeyError):
        preset("example9")
    assert set(BENCHMARKS) <= set(PRESETS)


def test_problem_and_rhs():
    spec = make_problem("example4a", 40)
    assert spec.dim == 2 and spec.n_modes == 39 and spec.axis_betas is not None
    assert np.all(benchmark_rhs(spec).data == 1.0)
    a = benchmark_rhs(spec, seed=7).data
    b = benchmark_rhs(spec, seed=7).data
    assert a.shape == (39, 39) and np.array_equal(a, b)
    # counter-based Philox stream, as the reference
    ref = np.random.Generator(np.random.Philox(7)).standard_normal((39, 39))
    assert np.array_equal(a, ref)


@pytest.mark.gpu
@pytest.mark.parametrize("case,n,tp", [("example1b", 320, (4, 0)), ("example2a", 40, (0, 0)),
                                       ("example2a", 40, (4, 3)), ("example3b", 12, (5, 0)),
                                       ("example4a", 40, ((4, 3), 0))])
def test_run_benchmark_matches_oracle(case, n, tp):
    from oracle import legpcg_port as orc
    from paper_2004_13961_b200 import run_benchmark
    rows = run_benchmark(case, n_list=[n], t_pairs=[tp])
    assert len(rows) == 1 and rows[0]["converged"]
    spec = make_problem(case, n)
    _, ro = orc.pcg_solve(spec, benchmark_rhs(spec).data, epsilon=BENCHMARKS[case]["epsilon"],
                          preconditioner=tp)
    assert abs(rows[0]["iterations"] - ro["iterations"]) <= 1
    assert rows[0]["rel_residual"] <= BENCHMARKS[case]["epsilon"]
