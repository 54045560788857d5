"""Matrix Market I/O and the CLI (§8(f) row 4): the writer is byte-identical
to the reference's (matrix_market.cc:12-38), the reader agrees with the
reference's on its files, and errors follow matrix_market.cc:46-93."""
import io
import os

import numpy as np
import pytest

from paper_2311_08316_b200.matrix_market import read_matrix_market, write_matrix_market


@pytest.fixture
def mat():
    rng = np.random.default_rng(3)
    a = rng.standard_normal((7, 5)) * 10.0 ** rng.integers(-20, 20, (7, 5))
    a[2, 3] = 0.0
    a[0, 0] = -0.0
    a[6, 4] = 1.0 / 3.0
    return np.asfortranarray(a)


@pytest.mark.parametrize("fmt", ["array", "coordinate"])
def test_round_trip(tmp_path, mat, fmt):
    p = str(tmp_path / "a.mtx")
    write_matrix_market(p, mat, fmt)
    back = read_matrix_market(p)
    assert back.shape == mat.shape and np.array_equal(back, mat)


@pytest.mark.parametrize("coordinate", [False, True])
def test_writer_byte_identical_to_reference(tmp_path, reference, mat, coordinate):
    ours, ref = str(tmp_path / "ours.mtx"), str(tmp_path / "ref.mtx")
    write_matrix_market(ours, mat, "coordinate" if coordinate else "array")
    reference.mm_write(ref, mat, coordinate)
    assert open(ours, "rb").read() == open(ref, "rb").read()
    assert np.array_equal(reference.mm_read(ours), read_matrix_market(ref))


def test_reader_comments_and_errors():
    text = "%%MatrixMarket matrix coordinate real general\n% a comment\n%\n3 2 2\n1 1 2.5\n3 2 -1\n"
    a = read_matrix_market(io.StringIO(text))
    assert a.shape == (3, 2) and a[0, 0] == 2.5 and a[2, 1] == -1.0 and np.count_nonzero(a) == 2
    bad = {
        "": "empty input",
        "%%MatrixMarket vector array real general\n1 1\n1\n": "not a Matrix Market matrix",
        "%%MatrixMarket matrix array real symmetric\n1 1\n1\n": "only real general",
        "%%MatrixMarket matrix array real general\n2 2\n1 2 3\n": "truncated array data",
        "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n": "out of range",
        "%%MatrixMarket matrix hyper real general\n2 2\n": "unknown format",
    }
    for t, msg in bad.items():
        with pytest.raises(RuntimeError, match=msg):
            read_matrix_market(io.StringIO(t))


def test_cli_gen_rejects_unknown_family():
    from paper_2311_08316_b200 import cli
    with pytest.raises(SystemExit):
        cli.main(["gen", "--matrix", "nope"])


def test_spectrum_values_match_reference_definition():
    from paper_2311_08316_b200.cli import spectrum_values
    s = spectrum_values("polynomial-decay", 100, 1e8)
    assert np.all(s[:10] == 1.0) and s[-1] == 1e-8 and np.all(np.diff(s) <= 0)
    st = spectrum_values("staircase", 8, 0)
    assert list(st) == [1.0, 1.0, 8e-10, 8e-10, 4e-10, 4e-10, 1e-10, 1e-10]
