"""CLI input parsing (no GPU): the covariate / outcome / assignment CSV
readers and their error contract (cli.py:49-121 of the reference)."""

import numpy as np
import pytest

from paper_2501_07642_b200 import cli
from paper_2501_07642_b200.errors import InputFormatError


def test_covariates_roundtrip_and_errors(tmp_path):
    p = tmp_path / "X.csv"
    p.write_text("a,b\n1,2\n3.5,-4e-3\n")
    cov, names = cli.parse_covariates(p)
    assert names == ["a", "b"] and np.array_equal(cov.values, [[1, 2], [3.5, -4e-3]])
    p.write_text("a,b\r\n1,2\r\n3,4\r\n")
    assert np.array_equal(cli.parse_covariates(p)[0].values, [[1, 2], [3, 4]])
    for body, msg in [("a,b\n1\n", "ragged row 1"), ("a,b\n1,x\n", "non-numeric cell at row 1, column 'b': 'x'"),
                      ("a,b\n1,nan\n", "non-finite value at row 1, column 'b'"), ("a,b\n", "no data rows"),
                      ("", "is empty")]:
        p.write_text(body)
        with pytest.raises(InputFormatError, match=msg):
            cli.parse_covariates(p)
    with pytest.raises(InputFormatError, match="cannot read"):
        cli.parse_covariates(tmp_path / "missing.csv")


def test_single_columns(tmp_path):
    p = tmp_path / "y.csv"
    p.write_text("y\n1.5\n-2\n")
    assert np.array_equal(cli.parse_outcomes(p), [1.5, -2.0])
    p.write_text("w\n1\n0\n1\n")
    w = cli.parse_assignment(p)
    assert w.dtype == np.int8 and w.tolist() == [1, 0, 1]
    p.write_text("w\n1\n2\n")
    with pytest.raises(InputFormatError, match="must be 0 or 1"):
        cli.parse_assignment(p)
    p.write_text("y\n1,2\n")
    with pytest.raises(InputFormatError, match="exactly one cell"):
        cli.parse_outcomes(p)


def test_parser_matches_reference_flags():
    ap = cli.build_parser()
    a = ap.parse_args(["generate", "--covariates", "X.csv", "--n-treated", "5", "--file", "p.csv"])
    assert (a.mode, a.accept_prob, a.max_draws, a.seed, a.precision, a.storage, a.out) == (
        "monte_carlo", 0.01, 100_000, 0, "exact", "keys", "p.csv")
    a = ap.parse_args(["test", "--pool", "p", "--outcomes", "y", "--observed", "w", "--find-fi", "--alpha", "0.1"])
    assert a.find_fi and a.alpha == 0.1
    a = ap.parse_args(["simulate", "--n", "10", "--k", "2"])
    assert (a.out_covariates, a.out_outcomes, a.out_assignment, a.tau, a.noise_sd) == ("X.csv", "y.csv", "w.csv", 1.0, 0.5)
