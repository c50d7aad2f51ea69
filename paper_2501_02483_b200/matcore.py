"""Scalar symmetric sparse matrices (lower-triangle CSC) and the arrowhead
generator — the input side of the path (reference matcore.py).

Heavy loops (pattern generation, diagonal sums, structure statistics) run in
the C++ host library; numpy only holds the arrays.  Matrix Market I/O is out
of scope (survey §2.1 row 7).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import check, i32p, i64p, f64p, lib, ptr
from .errors import MatrixFormatError

__all__ = ["SymmetricCsc", "from_coordinates", "ArrowheadSpec", "pattern_nnz_lower",
           "pattern_density_percent", "generate_arrowhead", "StructureStats",
           "structure_stats", "permute_symmetric"]


@dataclass(eq=False)
class SymmetricCsc:
    """Lower triangle of a symmetric matrix in CSC form (reference
    matcore.py:13-86): ``col_ptr`` int64[n+1], ``row_idx`` int32[nnz] strictly
    increasing per column and starting with the diagonal, ``values`` f64."""

    n: int
    col_ptr: np.ndarray
    row_idx: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.col_ptr[-1])

    @property
    def nnz_full(self) -> int:
        return 2 * self.nnz - self.n

    @property
    def density_percent(self) -> float:
        return 100.0 * self.nnz_full / (self.n * self.n)

    def diagonal(self) -> np.ndarray:
        return self.values[self.col_ptr[:-1]]

    def column(self, j: int):
        a, b = self.col_ptr[j], self.col_ptr[j + 1]
        return self.row_idx[a:b], self.values[a:b]

    def validate(self) -> None:
        n, cp, ri = self.n, self.col_ptr, self.row_idx
        if n < 1:
            raise ValueError("matrix order must be >= 1")
        if cp.shape != (n + 1,) or cp[0] != 0 or cp[-1] != ri.size or ri.size != self.values.size:
            raise ValueError("inconsistent CSC arrays")
        lens = np.diff(cp)
        if np.any(lens < 1):
            raise ValueError("col_ptr must be nondecreasing with nonempty columns")
        cols = np.repeat(np.arange(n), lens)
        first = ri[cp[:-1]]
        bad = np.flatnonzero(first != np.arange(n))
        if bad.size:
            raise ValueError(f"column {int(bad[0])} missing its diagonal entry")
        step = np.diff(ri.astype(np.int64))
        same = cols[1:] == cols[:-1]
        bad = np.flatnonzero(same & (step <= 0))
        if bad.size:
            raise ValueError(f"row indices not strictly increasing in column {int(cols[bad[0] + 1])}")
        last = ri[cp[1:] - 1]
        bad = np.flatnonzero(last >= n)
        if bad.size:
            raise ValueError(f"row index out of range in column {int(bad[0])}")
        if np.any(self.values[cp[:-1]] <= 0):
            raise ValueError("non-positive diagonal entry")

    def __eq__(self, other) -> bool:
        if not isinstance(other, SymmetricCsc):
            return NotImplemented
        return (self.n == other.n and np.array_equal(self.col_ptr, other.col_ptr)
                and np.array_equal(self.row_idx, other.row_idx)
                and np.array_equal(self.values, other.values))

    def to_dense(self) -> np.ndarray:
        if self.n > 20000:
            raise ValueError("refusing to densify a matrix this large")
        out = np.zeros((self.n, self.n))
        cols = np.repeat(np.arange(self.n), np.diff(self.col_ptr))
        out[cols, self.row_idx] = self.values
        out[self.row_idx, cols] = self.values
        return out


def _canonicalize(n, lo_r, lo_c, vals, sum_duplicates):
    """Sort lower coordinates by (col, row) stably and merge duplicates."""
    key = lo_c * np.int64(n) + lo_r
    order = np.argsort(key, kind="stable")
    key, vals = key[order], vals[order]
    if key.size:
        head = np.empty(key.size, dtype=bool)
        head[0] = True
        np.not_equal(key[1:], key[:-1], out=head[1:])
        if not head.all():
            if not sum_duplicates:
                raise MatrixFormatError("duplicate entries present")
            vals = np.add.reduceat(vals, np.flatnonzero(head))
            key = key[head]
    cols = key // n
    rows = key - cols * n
    col_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(cols, minlength=n), out=col_ptr[1:])
    return col_ptr, rows.astype(np.int32), np.ascontiguousarray(vals, dtype=np.float64)


def from_coordinates(n: int, rows, cols, vals, sum_duplicates: bool = True) -> SymmetricCsc:
    """Coordinates (either triangle) -> canonical SymmetricCsc
    (reference matcore.py:89-133, same error messages, 1-based columns)."""
    r = np.asarray(rows, dtype=np.int64)
    c = np.asarray(cols, dtype=np.int64)
    v = np.asarray(vals, dtype=np.float64)
    if r.size != c.size or r.size != v.size:
        raise ValueError("coordinate arrays must have equal length")
    if r.size and (min(r.min(), c.min()) < 0 or max(r.max(), c.max()) >= n):
        raise MatrixFormatError("coordinate index out of range")
    cp, ri, vv = _canonicalize(n, np.maximum(r, c), np.minimum(r, c), v, sum_duplicates)
    lens = np.diff(cp)
    if np.any(lens < 1):
        raise MatrixFormatError(f"missing diagonal entry in column {int(np.argmin(lens)) + 1}")
    first = ri[cp[:-1]]
    miss = first != np.arange(n)
    if np.any(miss):
        raise MatrixFormatError(f"missing diagonal entry in column {int(np.argmax(miss)) + 1}")
    nonpos = vv[cp[:-1]] <= 0
    if np.any(nonpos):
        raise MatrixFormatError(f"non-positive diagonal entry in column {int(np.argmax(nonpos)) + 1}")
    return SymmetricCsc(n, cp, ri, vv)


@dataclass(frozen=True)
class ArrowheadSpec:
    """Arrowhead shape (reference matcore.py:225-246): order n, half-band b of
    the leading block, t dense trailing rows, optional disjoint b-blocks."""

    n: int
    b: int
    t: int
    block_diagonal: bool = False
    seed: int = 0

    def __post_init__(self):
        if not (0 <= self.t < self.n):
            raise ValueError(f"need 0 <= t < n, got t={self.t}, n={self.n}")
        if not (0 <= self.b < self.n - self.t):
            raise ValueError(f"need 0 <= b < n - t, got b={self.b}, n-t={self.n - self.t}")
        if self.block_diagonal and self.b < 1:
            raise ValueError("block_diagonal needs b >= 1")


def pattern_nnz_lower(spec: ArrowheadSpec) -> int:
    """Closed-form stored count (reference matcore.py:249-260)."""
    nh = spec.n - spec.t
    if spec.block_diagonal:
        full, part = divmod(nh, spec.b)
        band = full * spec.b * (spec.b - 1) // 2 + part * (part - 1) // 2
    else:
        w = min(spec.b, nh - 1)
        band = w * (nh - w) + w * (w - 1) // 2
    return spec.n + band + spec.t * (nh + spec.n - 1) // 2


def pattern_density_percent(spec: ArrowheadSpec) -> float:
    return 100.0 * (2 * pattern_nnz_lower(spec) - spec.n) / (spec.n * spec.n)


def generate_arrowhead(spec: ArrowheadSpec, chunk: int = 1 << 26) -> SymmetricCsc:
    """Deterministic SPD arrowhead, bit-identical to reference
    matcore.py:269-317: PCG64 ``uniform(-1, 1)`` draws in CSC order (drawn in
    chunks; the concatenation equals one draw), diagonal = 1 + absolute row
    sum accumulated in CSC order (C++, same order as the two bincounts)."""
    n = spec.n
    cp = np.empty(n + 1, dtype=np.int64)
    check("tc_arrowhead_pattern", lib.tc_arrowhead_pattern(
        n, spec.b, spec.t, int(spec.block_diagonal), ptr(cp, i64p), None))
    nnz = int(cp[-1])
    if nnz != pattern_nnz_lower(spec):
        raise AssertionError("arrowhead pattern size mismatch")
    ri = np.empty(nnz, dtype=np.int32)
    check("tc_arrowhead_pattern", lib.tc_arrowhead_pattern(
        n, spec.b, spec.t, int(spec.block_diagonal), ptr(cp, i64p), ptr(ri, i32p)))
    vals = np.empty(nnz, dtype=np.float64)
    rng = np.random.default_rng(spec.seed)
    for lo in range(0, nnz, chunk):
        hi = min(nnz, lo + chunk)
        vals[lo:hi] = rng.uniform(-1.0, 1.0, size=hi - lo)
    check("tc_arrowhead_diag", lib.tc_arrowhead_diag(n, ptr(cp, i64p), ptr(ri, i32p), ptr(vals, f64p)))
    return SymmetricCsc(n, cp, ri, vals)


@dataclass(frozen=True)
class StructureStats:
    bandwidth: int
    thickness: int
    density_percent: float


def structure_stats(m: SymmetricCsc, dense_row_threshold: float = 0.5) -> StructureStats:
    """Trailing dense-row run and leading-block bandwidth (reference
    matcore.py:320-348), computed in C++."""
    bw = np.zeros(1, dtype=np.int64)
    th = np.zeros(1, dtype=np.int64)
    cp = _lib.i64arr(m.col_ptr)
    ri = _lib.i32arr(m.row_idx)
    check("tc_structure_stats", lib.tc_structure_stats(
        m.n, ptr(cp, i64p), ptr(ri, i32p), float(dense_row_threshold), ptr(bw, i64p), ptr(th, i64p)))
    return StructureStats(bandwidth=int(bw[0]), thickness=int(th[0]),
                          density_percent=m.density_percent)


def permute_symmetric(m: SymmetricCsc, p) -> SymmetricCsc:
    """B[p(i), p(j)] = A[i, j], re-canonicalised (reference matcore.py:351-366)."""
    fwd = np.asarray(getattr(p, "forward", p), dtype=np.int64)
    if fwd.shape != (m.n,):
        raise ValueError(f"permutation length {fwd.shape} does not match order {m.n}")
    hit = np.zeros(m.n, dtype=bool)
    hit[fwd] = True
    if not hit.all():
        raise ValueError("permutation is not a bijection")
    cols = np.repeat(np.arange(m.n, dtype=np.int64), np.diff(m.col_ptr))
    return from_coordinates(m.n, fwd[m.row_idx], fwd[cols], m.values, sum_duplicates=False)
