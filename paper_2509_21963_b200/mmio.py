"""MatrixMarket I/O (the input format before the path), restating
proj/src/testmat.cpp:134-355 — banner `%%MatrixMarket matrix {coordinate|array}
{real|integer} {general|symmetric}`, comment and blank lines skipped, 1-based coordinate
entries (duplicates, out-of-range indices and trailing tokens rejected), symmetric files
mirrored, array data column by column (lower triangle when symmetric). Coordinate files
become CSR handles, array files dense handles; errors carry the reference's
"path:line: what" messages as RuntimeError.
"""
from __future__ import annotations

import math

import numpy as np

from . import MatrixHandle


def _err(path, line, what):
    raise RuntimeError(f"{path}:{line}: {what}")


def _value(path, lineno, tok):
    try:
        v = float(tok)
    except ValueError:
        _err(path, lineno, f"malformed numeric value '{tok}'")
    if not math.isfinite(v):
        _err(path, lineno, "non-finite value")
    return v


def _content_lines(lines, start):
    """(lineno, text) of the lines after `start` that are neither blank nor comments."""
    for k in range(start, len(lines)):
        t = lines[k].lstrip(" \t\r")
        if not t or t.startswith("%"):
            continue
        yield k + 1, lines[k]


def read_matrix_market(path: str) -> MatrixHandle:
    try:
        with open(path) as fh:
            text = fh.read()
    except OSError:
        raise RuntimeError(f"cannot open '{path}'") from None
    if not text:
        _err(path, 1, "empty file")
    lines = text.split("\n")
    parts = lines[0].split()
    tag, obj, fmt, field, sym = (parts + [""] * 5)[:5]
    if tag != "%%MatrixMarket":
        _err(path, 1, "missing %%MatrixMarket banner")
    if obj.lower() != "matrix":
        _err(path, 1, f"unsupported object '{obj}'")
    if fmt.lower() not in ("coordinate", "array"):
        _err(path, 1, f"unsupported format '{fmt}'")
    if field.lower() not in ("real", "integer"):
        _err(path, 1, f"unsupported field '{field}'")
    if sym.lower() not in ("general", "symmetric"):
        _err(path, 1, f"unsupported symmetry '{sym}'")
    coordinate, symmetric = fmt.lower() == "coordinate", sym.lower() == "symmetric"
    it = _content_lines(lines, 1)
    try:
        lineno, size_line = next(it)
    except StopIteration:
        _err(path, len(lines), "missing size line")
    toks = size_line.split()
    if coordinate:
        try:
            rows, cols, declared = (int(x) for x in toks[:3])
        except ValueError:
            _err(path, lineno, "malformed coordinate size line")
        if len(toks) < 3 or rows < 0 or cols < 0 or declared < 0:
            _err(path, lineno, "malformed coordinate size line")
        if len(toks) > 3:
            _err(path, lineno, "trailing tokens on size line")
        if symmetric and rows != cols:
            _err(path, lineno, "symmetric matrix must be square")
        entries = {}
        for k in range(declared):
            try:
                lineno, line = next(it)
            except StopIteration:
                _err(path, len(lines), f"expected {declared} entries, file ended after {k}")
            t = line.split()
            if len(t) < 3:
                _err(path, lineno, "malformed coordinate entry")
            if len(t) > 3:
                _err(path, lineno, "trailing tokens on entry")
            try:
                i, j = int(t[0]), int(t[1])
            except ValueError:
                _err(path, lineno, "malformed coordinate entry")
            if i < 1 or i > rows or j < 1 or j > cols:
                _err(path, lineno, f"entry index ({i}, {j}) out of range")
            v = _value(path, lineno, t[2])
            for key in ((i - 1, j - 1),) + (((j - 1, i - 1),) if symmetric and i != j else ()):
                if key in entries:
                    _err(path, lineno, f"duplicate entry at ({key[0] + 1}, {key[1] + 1})")
                entries[key] = v
        for lineno, _ in it:
            _err(path, lineno, "unexpected data after the declared entries")
        keys = sorted(entries)
        indptr = np.zeros(rows + 1, dtype=np.int64)
        for (i, _j) in keys:
            indptr[i + 1] += 1
        indptr = np.cumsum(indptr)
        return MatrixHandle.sparse_csr(rows, cols, indptr, [j for _, j in keys], [entries[k] for k in keys])
    try:
        rows, cols = (int(x) for x in toks[:2])
    except ValueError:
        _err(path, lineno, "malformed array size line")
    if len(toks) < 2 or rows < 0 or cols < 0:
        _err(path, lineno, "malformed array size line")
    if len(toks) > 2:
        _err(path, lineno, "trailing tokens on size line")
    if symmetric and rows != cols:
        _err(path, lineno, "symmetric matrix must be square")
    expected = rows * (rows + 1) // 2 if symmetric else rows * cols
    data = []
    for lineno, line in it:
        for tok in line.split():
            if len(data) >= expected:
                _err(path, lineno, "unexpected data after the declared values")
            data.append(_value(path, lineno, tok))
    if len(data) < expected:
        _err(path, len(lines), f"expected {expected} values, found {len(data)}")
    out = np.zeros((rows, cols), order="F")
    k = 0
    for j in range(cols):
        for i in range(j if symmetric else 0, rows):
            out[i, j] = data[k]
            if symmetric:
                out[j, i] = data[k]
            k += 1
    return MatrixHandle.dense(out)


def write_matrix_market(path: str, a: MatrixHandle) -> None:
    try:
        fh = open(path, "w")
    except OSError:
        raise RuntimeError(f"cannot open '{path}' for writing") from None
    with fh:
        if a.is_sparse:
            rp, ci, v = a._csr
            fh.write("%%MatrixMarket matrix coordinate real general\n")
            fh.write(f"{a.rows} {a.cols} {v.size}\n")
            for i in range(a.rows):
                for p in range(rp[i], rp[i + 1]):
                    fh.write(f"{i + 1} {ci[p] + 1} {v[p]:.17g}\n")
        else:
            m = a.to_numpy()
            fh.write("%%MatrixMarket matrix array real general\n")
            fh.write(f"{m.shape[0]} {m.shape[1]}\n")
            for x in m.ravel(order="F"):
                fh.write(f"{x:.17g}\n")
