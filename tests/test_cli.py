"""SPEC cmd_solve through paper_2506_08355_b200.cli: argument and ingestion
errors and the canonical JSON report on CPU; the SPEC's examples (PAPER Tables 2/3) on the GPU."""
import csv
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_cli(*args, cwd=None):
    return subprocess.run([sys.executable, "-m", "paper_2506_08355_b200.cli", *args], cwd=cwd or ROOT,
                          capture_output=True, text=True, timeout=600)


def test_exit_1_on_argument_errors():
    assert run_cli("solve").returncode == 1                      # no problem source
    assert run_cli("solve", "--problem", "t0", "--k-file", "a.mtx", "--m-file", "b.mtx").returncode == 1
    assert run_cli("solve", "--problem", "nope").returncode == 1
    assert run_cli("bogus").returncode == 1


def test_exit_2_on_ingestion_error(tmp_path):
    bad = tmp_path / "bad.mtx"
    bad.write_text("%%MatrixMarket matrix coordinate real general\n3 3 2\n1 1 1.0\n")  # truncated
    r = run_cli("solve", "--k-file", str(bad), "--m-file", str(bad))
    assert r.returncode == 2, r.stderr
    assert "ingestion error" in r.stderr


def test_report_json_round_trips_byte_identical():
    from paper_2506_08355_b200.cli import dumps
    rep = {"eigenvalues": [9.849886676638346e-06, 0.1 + 0.2], "b": {"z": 1, "a": None}, "converged": True}
    s = dumps(rep)
    assert dumps(json.loads(s)) == s
    assert json.loads(s)["eigenvalues"][1] == 0.1 + 0.2  # real64-exact


@pytest.mark.gpu
def test_table2_example(tmp_path):
    out, hist = tmp_path / "r.json", tmp_path / "h.csv"
    r = run_cli("solve", "--problem", "t0", "--n", "1000", "--nev", "10", "--nb", "10", "--tol", "1e-10",
                "--out", str(out), "--history", str(hist))
    assert r.returncode == 0, r.stderr
    assert "9.849886676638E-06" in r.stdout  # PAPER Table 2, lambda_1
    rep = json.loads(out.read_text())
    assert rep["converged"] and len(rep["eigenvalues"]) == 10
    assert all(x <= y for x, y in zip(rep["eigenvalues"], rep["eigenvalues"][1:]))
    assert max(rep["residuals"]) <= 1e-10
    rows = list(csv.reader(hist.open()))[1:]
    assert len(rows) == rep["iterations"] * 10


@pytest.mark.gpu
def test_table3_example():
    r = run_cli("solve", "--problem", "tm1", "--n", "1000", "--nev", "10", "--tol", "1e-10")
    assert r.returncode == 0, r.stderr
    assert "3.943890108210E-05" in r.stdout  # PAPER Table 3, lambda_1


@pytest.mark.gpu
def test_full_positive_spectrum_and_matrix_market(tmp_path):
    # SPEC's "full positive spectrum" example: the UNMODIFIED reference does not converge on it
    # either (30 of 49 pairs after 500 iterations, measured with oracle/_ref) -- exit 3 with the
    # report written is the reference-equivalent outcome
    out0 = tmp_path / "full.json"
    r = run_cli("solve", "--problem", "t0", "--n", "50", "--nev", "49", "--tol", "1e-8", "--out", str(out0))
    assert r.returncode == 3, r.stderr
    assert json.loads(out0.read_text())["converged"] is False
    # the same T(0) from Matrix Market files
    from paper_2506_08355_b200 import problems as P
    t = P.t_matrix(200, 0.0)
    path = tmp_path / "t.mtx"
    with path.open("w") as f:
        f.write(f"%%MatrixMarket matrix coordinate real general\n{t.n} {t.n} {t.nnz}\n")
        for i in range(t.n):
            for k in range(t.rowptr[i], t.rowptr[i + 1]):
                f.write(f"{i + 1} {int(t.colidx[k]) + 1} {float(t.vals[k])!r}\n")
    out = tmp_path / "r.json"
    r = run_cli("solve", "--k-file", str(path), "--m-file", str(path), "--nev", "5", "--tol", "1e-10",
                "--out", str(out))
    assert r.returncode == 0, r.stderr
    lam = json.loads(out.read_text())["eigenvalues"]
    import numpy as np
    assert np.allclose(lam, P.t_eigenvalues(200, 5), rtol=1e-11)
