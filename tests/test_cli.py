"""CLI (the reference's cli.py contract) on the GPU path: config validation and exit
codes on CPU, solve / table / bench-matvec on the B200."""

import json

import pytest

from paper_2004_13961_b200.cli import main, t_pairs


def _cfg(tmp_path, obj):
    p = tmp_path / "cfg.json"
    p.write_text(json.dumps(obj))
    return str(p)


@pytest.mark.parametrize("obj", [{"n": 16}, {"example": "example2a", "coefficients": {"beta": 1}, "n": 8},
                                 {"example": "nope", "n": 8}, {"example": "example2a"},
                                 {"example": "example2a", "n": 8, "bogus": 1},
                                 {"coefficients": {"beta": 1.0}, "n": 8}])
def test_solve_config_errors_exit_1(tmp_path, obj):
    assert main(["solve", "--config", _cfg(tmp_path, obj)]) == 1


def test_usage_errors_exit_1(tmp_path):
    assert main(["nosuchcommand"]) == 1
    assert main(["solve", "--config", str(tmp_path / "missing.json")]) == 1
    assert main(["table", "--example", "example9"]) == 1
    assert main(["table", "--example", "example2a", "--n", ""]) == 1
    assert main(["bench-matvec", "--dim", "2", "--n", "16", "--reps", "2"]) == 1
    assert main(["bench-matvec", "--dim", "2", "--n", "16", "--preset", "example3a"]) == 1
    assert main(["rank", "--preset", "expx", "--which", "A", "--n", "16"]) == 1
    assert t_pairs("6,2;4/3,0") == [(6, 2), ((4, 3), 0)]


@pytest.mark.gpu
def test_solve_table_benchmatvec(tmp_path, capsys):
    out = tmp_path / "res.json"
    code = main(["solve", "--config", _cfg(tmp_path, {"example": "example2a", "n": 40, "t1": 4, "t2": 3}),
                 "--out", str(out)])
    assert code == 0
    res = json.loads(out.read_text())
    assert res["converged"] and res["N"] == 40 and res["rel_residual"] <= 1e-7
    code = main(["solve", "--config", _cfg(tmp_path, {"coefficients": {"beta": 2.0, "alpha": 1.0},
                                                       "dim": 3, "n": 12, "t1": 2, "t2": 2})])
    assert code == 0
    assert main(["table", "--example", "example3b", "--n", "12", "--t", "0,0;5,0",
                 "--format", "json", "--out", str(tmp_path / "t.json")]) == 0
    rows = json.loads((tmp_path / "t.json").read_text())
    assert len(rows) == 2 and all(r["converged"] for r in rows)
    assert main(["bench-matvec", "--dim", "2", "--n", "32,64", "--preset", "example2a",
                 "--reps", "3", "--format", "csv"]) == 0
    assert "d,N,op,time_s" in capsys.readouterr().out
    # non-convergence: exit code 2
    assert main(["solve", "--config", _cfg(tmp_path, {"example": "example2a", "n": 40, "kmax": 1,
                                                       "epsilon": 1e-14})]) == 2
