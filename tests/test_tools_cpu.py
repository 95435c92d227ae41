"""CPU checks of the measurement helpers: bench.py's reference for the error column and the
paper-experiment tool's command line (PAPER.md:353-354 standards, SPEC's CSV / JSON schema)."""
import json
import os
import sys
from fractions import Fraction

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))


def test_exact_rows_is_the_correctly_rounded_product():
    import bench

    rng = np.random.default_rng(3)
    for trial in range(4):
        P = int(rng.integers(1, 400))
        A = rng.standard_normal((2, P)) * 10.0 ** rng.integers(-8, 8, (2, P))
        B = rng.standard_normal((P, 5)) * 10.0 ** rng.integers(-8, 8, (P, 5))
        X = bench.exact_rows(A, B)
        for r in range(2):
            for j in range(5):
                ex = sum(Fraction(float(A[r, k])) * Fraction(float(B[k, j])) for k in range(P))
                # Dot2's bound: u |x| + (P u)^2 sum |a b|; in practice the correctly rounded value
                bound = 2.0 ** -53 * abs(float(ex)) + (P * 2.0 ** -53) ** 2 * float(np.abs(A[r] * B[:, j]).sum())
                assert abs(X[r, j] - float(ex)) <= bound, (trial, r, j)
    # cancellation: the sum is exactly 1 although every partial sum is huge
    A = np.array([[1e300 / 1e290, 1.0, -1e300 / 1e290]])
    B = np.array([[1e10], [1.0], [1e10]])
    assert bench.exact_rows(A, B)[0, 0] == 1.0


def test_paper_experiment_cli_defaults_and_errors():
    import paper_experiment as pe

    a = pe.parse_args([])
    assert (a.order, a.repeats, a.seed, a.sizes, a.methods, a.format) == (400, 10, 42, [400], None, "table")
    a = pe.parse_args(["-O", "200", "-R", "3", "--methods", "NaivStandard,WinogradScaled", "--format", "csv"])
    assert (a.sizes, a.repeats, a.methods) == ([200], 3, ["NaivStandard", "WinogradScaled"])
    for bad in (["-O", "abc"], ["-O", "0"], ["-R", "-1"], ["--methods", "Foo"], ["--format", "xml"], ["--bogus"]):
        with pytest.raises(SystemExit) as e:
            pe.parse_args(bad)
        assert e.value.code == 2, bad


def test_paper_experiment_csv_schema():
    import paper_experiment as pe

    rows = [{"n": 4, "method": "NaivKahan", "seconds": 0.25, "deviation": None},
            {"n": 4, "method": "NaivStandard", "seconds": 0.125, "deviation": 1.23456789e-10}]
    lines = pe.render_csv(rows).splitlines()
    assert lines[0] == "method,seconds,deviation"
    assert lines[1] == "NaivKahan,0.25," and len(lines) == 3
    m, t, d = lines[2].split(",")
    assert (m, float(t), float(d)) == ("NaivStandard", 0.125, 1.23456789e-10)
    table = pe.render_table(rows, 4, 10, {}, {})
    assert "C = A*(8A)" in table and "N := NaivKahan" in table and "0.0000000001" in table
    json.dumps({"results": rows})
