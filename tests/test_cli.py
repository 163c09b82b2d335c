"""The command-line front end (python -m paper_1710_01048_b200): JSON rule export with the
paper's constants, exit-code contract (0 / 2 / 4), counts, and (GPU) assembly
with MatrixMarket output."""
import json
import subprocess
import sys

import numpy as np
import pytest

from paper_1710_01048_b200.__main__ import main


def test_derive_rules_paper_constants(tmp_path, capsys):
    out = tmp_path / "r.json"
    assert main(["derive-rules", "--degree", "2", "--kind", "mass", "--out", str(out)]) == 0
    doc = json.loads(out.read_text())
    interior = next(e for e in doc if e["class"] == "interior")
    assert abs(interior["nodes"][0] - 0.71241440095955149482) < 1e-15            # eq:WQquadratic
    assert main(["derive-rules", "--degree", "3", "--kind", "stiffness"]) == 0
    doc = json.loads(capsys.readouterr().out)
    interior = next(e for e in doc if e["class"] == "interior")
    assert abs(interior["nodes"][0] - 0.24033518882038592858) < 1e-15            # P:419 (tau_1)


def test_exit_codes(capsys):
    assert main(["derive-rules", "--degree", "4"]) == 4                         # unsupported degree
    assert main(["nonsense"]) == 4                                               # config error
    assert main(["derive-rules", "--degree", "3", "--tol", "1e-40"]) == 2        # residual above tolerance
    capsys.readouterr()


def test_counts_command(capsys):
    assert main(["counts", "--degree", "3", "--dim", "2", "--mesh", "20"]) == 0
    doc = json.loads(capsys.readouterr().out)
    assert doc["mass"]["newton_cotes"] > doc["mass"]["gaussian"] > 0


@pytest.mark.gpu
def test_assemble_command_writes_matrix_market(tmp_path):
    prefix = str(tmp_path / "m")
    r = subprocess.run([sys.executable, "-m", "paper_1710_01048_b200", "assemble", "--degree", "2", "--dim", "1",
                        "--mesh", "6", "--coef", "const", "--layout", "csr", "--mtx", prefix],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    lines = open(prefix + "_mass.mtx").read().splitlines()
    n, _, nnz = map(int, lines[1].split())
    A = np.zeros((n, n))
    for l in lines[2:]:
        i, j, v = l.split()
        A[int(i) - 1, int(j) - 1] = float(v)
    assert n == 8 and nnz == len(lines) - 2
    assert np.allclose(A, A.T, atol=1e-15) and abs(A.sum() - 1.0) < 1e-14      # c = 1: symmetric, sum = |[0,1]|


@pytest.mark.gpu
def test_eigen_command(capsys):
    assert main(["eigen", "--degree", "3", "--dim", "1", "--mesh", "64", "--count", "5"]) == 0
    doc = json.loads(capsys.readouterr().out)
    assert doc["dofs"] == 65 and len(doc["rel_err"]) == 5
    assert all(0 <= e < 1e-5 for e in doc["rel_err"])             # Rayleigh-Ritz: from above
    assert abs(doc["exact"][0] - np.pi ** 2) < 1e-12
