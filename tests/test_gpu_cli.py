"""The CLI (paper_2311_08316_b200/cli.py, §8(f) row 4) end to end on the GPU:
factor writes Q/R as Matrix Market and a 1-based pivot list that match the
reference algorithm (the oracle), profile prints the phase table."""
import numpy as np
import pytest

from paper_2311_08316_b200.matrix_market import read_matrix_market, write_matrix_market

pytestmark = pytest.mark.gpu


def test_cli_factor_matches_reference_algorithm(cuda, oracle, tmp_path, capsys):
    from paper_2311_08316_b200 import cli
    a = oracle.gen_gaussian(800, 40, 5)
    inp = str(tmp_path / "a.mtx")
    write_matrix_market(inp, a, "coordinate")
    pre = str(tmp_path / "out")
    assert cli.main(["--seed", "3", "factor", "--in", inp, "--out-prefix", pre, "--nnz", "8"]) == 0
    out = capsys.readouterr().out
    assert "validation pass" in out
    q, r = read_matrix_market(pre + "_Q.mtx"), read_matrix_market(pre + "_R.mtx")
    j = np.loadtxt(pre + "_J.txt", dtype=np.int64)
    ref = oracle.cqrrpt(a, gamma=1.25, nnz=8, seed=3)
    assert np.array_equal(j - 1, ref.pivots)  # 1-based on disk (cqrrpt_cli.cc:199)
    assert q.shape == (800, ref.k) and r.shape == (ref.k, 40)
    assert np.linalg.norm(a[:, j - 1] - q @ r) <= 1e-13 * np.linalg.norm(a)


def test_cli_gen_and_profile(cuda, tmp_path, capsys):
    from paper_2311_08316_b200 import cli
    p = str(tmp_path / "k.mtx")
    assert cli.main(["gen", "--matrix", "kahan", "--n", "16", "--out", p]) == 0
    k = read_matrix_market(p)
    assert k.shape == (16, 16) and k[0, 0] == 1.0 and np.all(np.tril(k, -1) == 0)
    csv = str(tmp_path / "prof.csv")
    assert cli.main(["profile", "--matrix", "polynomial-decay", "--m", "4096", "--n", "128", "--nnz", "8",
                     "--runs", "2", "--out", csv]) == 0
    out = capsys.readouterr().out
    assert "qrcp" in out and "detected rank k=" in out
    rows = open(csv).read().splitlines()
    assert rows[0].startswith("experiment,") and any(",time_total," in r for r in rows)
