"""Matrix Market coordinate files (host-side CRS build).

Same contract as pkg/src/levelmpk/mmio.py:22-109 -- coordinate format only;
real / integer / pattern fields; general or symmetric storage; square
matrices; symmetric storage is expanded, pattern entries become 1.0,
duplicates are summed (via CsrMatrix.from_triplets) and every error is a
MatrixMarketError naming the file and line.  File I/O is outside the GPU path
(SURVEY.md section 2, row 10).
"""

import numpy as np

from .csr import CsrMatrix

_FIELDS = {"real": 3, "integer": 3, "pattern": 2}
_SYMMETRIES = ("general", "symmetric")


class MatrixMarketError(ValueError):
    """Malformed Matrix Market input; message carries the offending line number."""


class _Reader:
    def __init__(self, path):
        self.path = str(path)
        with open(self.path, "r") as fh:
            self.lines = fh.read().splitlines()

    def error(self, lineno, msg):
        return MatrixMarketError(f"{self.path}:{lineno}: {msg}")

    def data_lines(self, start):
        """(1-based line number, stripped text) of non-comment, non-blank lines."""
        for idx in range(start, len(self.lines)):
            text = self.lines[idx].strip()
            if text and not text.startswith("%"):
                yield idx + 1, text


def _parse_header(rd: _Reader):
    if not rd.lines:
        raise rd.error(1, "empty file")
    tokens = rd.lines[0].split()
    if len(tokens) != 5 or tokens[0] != "%%MatrixMarket":
        raise rd.error(1, f"malformed header {rd.lines[0].strip()!r}")
    obj, fmt, field, symmetry = (t.lower() for t in tokens[1:])
    if (obj, fmt) != ("matrix", "coordinate"):
        raise rd.error(1, f"only 'matrix coordinate' files are supported, got {obj} {fmt}")
    if field not in _FIELDS:
        raise rd.error(1, f"unsupported field {field!r} (real, integer, or pattern)")
    if symmetry not in _SYMMETRIES:
        raise rd.error(1, f"unsupported symmetry {symmetry!r} (general or symmetric)")
    return field, symmetry


def load_matrix_market(path, device=False) -> CsrMatrix:
    """Read a coordinate-format Matrix Market file into a canonical CsrMatrix.

    device=True builds the CRS in HBM (lmpk_csr_from_triplets, bit-exact with
    the host build); parsing stays on the host (mmio.py:22-96)."""
    rd = _Reader(path)
    field, symmetry = _parse_header(rd)
    entries = rd.data_lines(1)
    try:
        size_no, size_text = next(entries)
    except StopIteration:
        raise rd.error(len(rd.lines), "missing size line") from None
    dims = size_text.split()
    if len(dims) != 3:
        raise rd.error(size_no, f"size line must be 'rows cols nnz', got {size_text!r}")
    try:
        n_rows, n_cols, n_entries = map(int, dims)
    except ValueError:
        raise rd.error(size_no, f"non-integer size line {size_text!r}") from None
    if n_rows != n_cols:
        raise MatrixMarketError(
            f"{rd.path}: matrix is {n_rows}x{n_cols}; only square matrices are supported")
    need = _FIELDS[field]
    ijv = np.empty((n_entries, 3), dtype=np.float64)
    count = 0
    for lineno, text in entries:
        if count >= n_entries:
            raise rd.error(lineno, f"more than the declared {n_entries} entries")
        parts = text.split()
        if len(parts) < need:
            raise rd.error(lineno, f"expected {need} fields, got {len(parts)}")
        try:
            i, j = int(parts[0]), int(parts[1])
            v = float(parts[2]) if need == 3 else 1.0
        except ValueError:
            raise rd.error(lineno, f"could not parse entry {text!r}") from None
        if not (1 <= i <= n_rows and 1 <= j <= n_cols):
            raise rd.error(lineno, f"index ({i}, {j}) out of range for {n_rows}x{n_cols} matrix")
        ijv[count] = (i - 1, j - 1, v)
        count += 1
    if count != n_entries:
        raise rd.error(len(rd.lines), f"expected {n_entries} entries, found {count}")
    r = ijv[:, 0].astype(np.int64)
    c = ijv[:, 1].astype(np.int64)
    v = ijv[:, 2]
    if symmetry == "symmetric":
        mirror = r != c
        r, c, v = (np.concatenate([r, c[mirror]]), np.concatenate([c, r[mirror]]),
                   np.concatenate([v, v[mirror]]))
    if device:
        import torch

        r, c, v = (torch.from_numpy(np.ascontiguousarray(t)).cuda() for t in (r, c, v))
    return CsrMatrix.from_triplets(n_rows, r, c, v)


def save_matrix_market(a: CsrMatrix, path, comment=None):
    """Write a CsrMatrix as 'coordinate real general' with 1-based indices."""
    rows, cols, vals = a.to_triplets()
    out = ["%%MatrixMarket matrix coordinate real general"]
    if comment:
        out += [f"% {line}" for line in str(comment).splitlines()]
    out.append(f"{a.n_rows} {a.n_rows} {a.n_nz}")
    out += [f"{r + 1} {c + 1} {float(v)!r}" for r, c, v in zip(rows, cols, vals)]
    with open(str(path), "w") as fh:
        fh.write("\n".join(out) + "\n")
