"""Matrix text format (SPEC.md cli module, ``MatrixFile``; SURVEY §8f rank 3 — the data
format either side of the hot path; the reference package itself has no file I/O).

    gf2e-mat v1 e=<e> f=<hex> rows=<m> cols=<n> repr=<packed|sliced>
    <row 0: entries as lowercase hex integers < 2^e, separated by single spaces>
    ...
    (trailing newline)

``repr`` records which representation the matrix was saved from (``PackedMatrix`` → packed,
``SlicedMatrix`` → sliced) and selects the type ``parse``/``load_matrix`` return; the body is
always the element values.  ``parse(serialize(A)) == A`` for every matrix; canonical files
round-trip byte for byte.  Host-side plumbing: conversions to and from device matrices go
through ``PackedMatrix.from_array`` / ``to_array`` (device kernels); the text itself is
formatted and parsed with numpy on the host.
"""

from __future__ import annotations

import re

import numpy as np

from .gf2e import field_new
from .mat_packed import PackedMatrix
from .mat_sliced import SlicedMatrix, cling, slice_packed

_HEADER = re.compile(r"^gf2e-mat v1 e=(\d+) f=([0-9a-f]+) rows=(\d+) cols=(\d+) repr=(packed|sliced)$")


def serialize(A) -> str:
    """Canonical text of a PackedMatrix or SlicedMatrix."""
    if isinstance(A, SlicedMatrix):
        rep, P = "sliced", cling(A)
    elif isinstance(A, PackedMatrix):
        rep, P = "packed", A
    else:
        raise TypeError(f"expected PackedMatrix or SlicedMatrix, got {type(A).__name__}")
    ctx = P.ctx
    lines = [f"gf2e-mat v1 e={ctx.e} f={ctx.f:x} rows={P.nrows} cols={P.ncols} repr={rep}"]
    if P.nrows:
        arr = P.to_array() if P.ncols else np.zeros((P.nrows, 0), dtype=np.uint16)
        hexes = np.char.mod("%x", arr.astype(np.int64)) if P.ncols else None
        for i in range(P.nrows):
            lines.append(" ".join(hexes[i].tolist()) if P.ncols else "")
    return "\n".join(lines) + "\n"


def parse(text: str):
    """Inverse of ``serialize``; raises ValueError on a malformed header or body, an entry
    out of range, or dimensions that do not match the header."""
    if not text.endswith("\n"):
        raise ValueError("matrix file must end with a newline")
    lines = text[:-1].split("\n")
    m = _HEADER.match(lines[0])
    if not m:
        raise ValueError(f"bad matrix file header: {lines[0][:80]!r}")
    e, f, rows, cols, rep = int(m.group(1)), int(m.group(2), 16), int(m.group(3)), int(m.group(4)), m.group(5)
    ctx = field_new(e, f)
    body = lines[1:]
    if len(body) != rows:
        raise ValueError(f"header says {rows} rows, body has {len(body)}")
    arr = np.zeros((rows, cols), dtype=np.uint16)
    for i, line in enumerate(body):
        toks = line.split(" ") if line else []
        if len(toks) != cols:
            raise ValueError(f"row {i}: expected {cols} entries, got {len(toks)}")
        for j, t in enumerate(toks):
            if not t or not re.fullmatch(r"[0-9a-f]+", t):
                raise ValueError(f"row {i}: entry {j} is not a lowercase hex integer: {t!r}")
            v = int(t, 16)
            if v >= ctx.order:
                raise ValueError(f"row {i}: entry {j} = {v} out of range for GF(2^{e})")
            arr[i, j] = v
    P = PackedMatrix.from_array(ctx, arr) if rows and cols else PackedMatrix(ctx, rows, cols)
    return slice_packed(P) if rep == "sliced" else P


def save_matrix(path, A) -> None:
    with open(path, "w", newline="\n") as fh:
        fh.write(serialize(A))


def load_matrix(path):
    with open(path, "r", newline="\n") as fh:
        return parse(fh.read())


__all__ = ["serialize", "parse", "save_matrix", "load_matrix"]
