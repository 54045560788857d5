"""Matrix Market I/O with the reference's conventions (matrix_market.cc:12-93):
real general matrices, `array` (column-major values) or `coordinate`
(1-based `i j v` in column-major order, zeros omitted), 17 significant digits
(`os.precision(17)` on the default float format == printf "%.17g")."""
from __future__ import annotations

import io
from typing import TextIO, Union

import numpy as np

PathOrFile = Union[str, TextIO]


def _fmt(v: float) -> str:
    return format(float(v), ".17g")


def write_matrix_market(dst: PathOrFile, m, fmt: str = "array") -> None:
    """write_matrix_market (matrix_market.cc:12-38)."""
    a = np.asarray(m, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError("write_matrix_market: expected a matrix")
    if fmt not in ("array", "coordinate"):
        raise ValueError("write_matrix_market: format must be 'array' or 'coordinate'")
    rows, cols = a.shape
    out = io.StringIO()
    if fmt == "array":
        out.write("%%MatrixMarket matrix array real general\n")
        out.write(f"{rows} {cols}\n")
        for v in a.flatten(order="F"):
            out.write(_fmt(v) + "\n")
    else:
        flat = a.flatten(order="F")
        nz = np.flatnonzero(flat != 0.0)
        out.write("%%MatrixMarket matrix coordinate real general\n")
        out.write(f"{rows} {cols} {nz.size}\n")
        for e in nz:
            j, i = divmod(int(e), rows)
            out.write(f"{i + 1} {j + 1} {_fmt(flat[e])}\n")
    text = out.getvalue()
    if isinstance(dst, str):
        try:
            with open(dst, "w") as f:
                f.write(text)
        except OSError as e:
            raise RuntimeError(f"write_matrix_market: cannot open {dst}") from e
    else:
        dst.write(text)


def read_matrix_market(src: PathOrFile) -> np.ndarray:
    """read_matrix_market (matrix_market.cc:46-93) -> column-major float64."""
    if isinstance(src, str):
        try:
            with open(src) as f:
                return read_matrix_market(f)
        except OSError as e:
            raise RuntimeError(f"read_matrix_market: cannot open {src}") from e
    header = src.readline()
    if not header:
        raise RuntimeError("read_matrix_market: empty input")
    parts = header.split()
    parts += [""] * (5 - len(parts))
    banner, obj, form, field, symmetry = parts[:5]
    if banner != "%%MatrixMarket" or obj.lower() != "matrix":
        raise RuntimeError("read_matrix_market: not a Matrix Market matrix")
    form = form.lower()
    if field.lower() != "real" or symmetry.lower() != "general":
        raise RuntimeError("read_matrix_market: only real general matrices are supported")
    line = src.readline()
    while line and (not line.strip() or line.startswith("%")):
        line = src.readline()
    tokens = src.read().split()
    if form == "array":
        try:
            rows, cols = (int(t) for t in line.split()[:2])
        except ValueError as e:
            raise RuntimeError("read_matrix_market: bad size line") from e
        if len(tokens) < rows * cols:
            raise RuntimeError("read_matrix_market: truncated array data")
        vals = np.array(tokens[: rows * cols], dtype=np.float64)
        return vals.reshape((rows, cols), order="F")
    if form == "coordinate":
        try:
            rows, cols, nnz = (int(t) for t in line.split()[:3])
        except ValueError as e:
            raise RuntimeError("read_matrix_market: bad size line") from e
        if len(tokens) < 3 * nnz:
            raise RuntimeError("read_matrix_market: truncated coordinate data")
        m = np.zeros((rows, cols), order="F")
        for t in range(nnz):
            i, j, v = int(tokens[3 * t]), int(tokens[3 * t + 1]), float(tokens[3 * t + 2])
            if i < 1 or i > rows or j < 1 or j > cols:
                raise RuntimeError("read_matrix_market: entry index out of range")
            m[i - 1, j - 1] = v
        return m
    raise RuntimeError(f"read_matrix_market: unknown format {form}")
