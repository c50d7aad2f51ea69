"""Fill-reducing orderings and exact fill counts (reference ordering.py).

RCM, adaptable nested dissection and the elimination-tree fill count run in
the C++ host library and are bit-exact with the reference (same tie-breaks);
selection keeps the identity unless a candidate is strictly smaller.
"""

from __future__ import annotations

import heapq
from dataclasses import dataclass

import numpy as np

from ._lib import check, i32p, i64p, lib, ptr, i64arr, i32arr
from .matcore import StructureStats, SymmetricCsc

__all__ = ["Permutation", "FillReport", "rcm", "min_degree", "adaptable_nd",
           "symbolic_fill_count", "select_ordering"]


@dataclass(eq=False)
class Permutation:
    """forward[old] = new, inverse[new] = old (reference ordering.py:18-68)."""

    forward: np.ndarray
    inverse: np.ndarray

    @classmethod
    def identity(cls, n: int) -> "Permutation":
        f = np.arange(n, dtype=np.int64)
        return cls(f, f.copy())

    @classmethod
    def from_forward(cls, forward) -> "Permutation":
        f = np.asarray(forward, dtype=np.int64)
        n = f.size
        if n and (f.min() < 0 or f.max() >= n):
            raise ValueError("forward map has out-of-range entries")
        inv = np.full(n, -1, dtype=np.int64)
        inv[f] = np.arange(n, dtype=np.int64)
        if n and inv.min() < 0:
            raise ValueError("forward map is not a bijection")
        return cls(f, inv)

    @property
    def n(self) -> int:
        return self.forward.size

    def is_identity(self) -> bool:
        return bool(np.array_equal(self.forward, np.arange(self.n)))

    def compose(self, other: "Permutation") -> "Permutation":
        """self o other: ``other`` applied first."""
        return Permutation.from_forward(self.forward[other.forward])

    def to_text(self) -> str:
        return " ".join(map(str, self.forward.tolist()))

    @classmethod
    def from_text(cls, text: str) -> "Permutation":
        return cls.from_forward([int(x) for x in text.split()])

    def __eq__(self, other) -> bool:
        if not isinstance(other, Permutation):
            return NotImplemented
        return bool(np.array_equal(self.forward, other.forward))


@dataclass(frozen=True)
class FillReport:
    nnz_original: int
    nnz_factor: int

    @property
    def fill_in(self) -> int:
        return self.nnz_factor - self.nnz_original


def _csc(m: SymmetricCsc):
    return i64arr(m.col_ptr), i32arr(m.row_idx)


def rcm(m: SymmetricCsc, pinned_tail: int = 0) -> Permutation:
    """Partial reverse Cuthill-McKee on the leading n - pinned_tail vertices
    (reference ordering.py:134-170)."""
    if not (0 <= pinned_tail <= m.n):
        raise ValueError(f"pinned_tail must be in [0, {m.n}]")
    cp, ri = _csc(m)
    fwd = np.empty(m.n, dtype=np.int64)
    check("tc_rcm", lib.tc_rcm(m.n, ptr(cp, i64p), ptr(ri, i32p), int(pinned_tail), ptr(fwd, i64p)))
    return Permutation.from_forward(fwd)


def adaptable_nd(m: SymmetricCsc, stats: StructureStats, max_levels: int = 8) -> Permutation:
    """Arrowhead nested dissection with bandwidth-wide separators moved ahead
    of the tail (reference ordering.py:209-236)."""
    fwd = np.empty(m.n, dtype=np.int64)
    check("tc_adaptable_nd", lib.tc_adaptable_nd(m.n, int(stats.bandwidth), int(stats.thickness),
                                                 int(max_levels), ptr(fwd, i64p)))
    return Permutation.from_forward(fwd)


def min_degree(m: SymmetricCsc) -> Permutation:
    """Exact greedy minimum degree (reference ordering.py:173-206).  Optional
    ordering, off the auto policy; host-only quotient-graph
    elimination with ties broken by the smallest index."""
    n = m.n
    cols = np.repeat(np.arange(n, dtype=np.int64), np.diff(m.col_ptr))
    rows = m.row_idx.astype(np.int64)
    off = rows != cols
    nbr = [set() for _ in range(n)]
    for a, b in zip(rows[off].tolist(), cols[off].tolist()):
        nbr[a].add(b)
        nbr[b].add(a)
    alive = [True] * n
    heap = [(len(nbr[v]), v) for v in range(n)]
    heapq.heapify(heap)
    fwd = np.empty(n, dtype=np.int64)
    for step in range(n):
        while True:
            d, v = heapq.heappop(heap)
            if alive[v] and d == len(nbr[v]):
                break
        alive[v] = False
        fwd[v] = step
        clique = sorted(nbr[v])
        for w in clique:
            nbr[w].discard(v)
        for i, a in enumerate(clique):
            na = nbr[a]
            for b in clique[i + 1:]:
                if b not in na:
                    na.add(b)
                    nbr[b].add(a)
        for w in clique:
            heapq.heappush(heap, (len(nbr[w]), w))
        nbr[v] = set()
    return Permutation.from_forward(fwd)


def symbolic_fill_count(m: SymmetricCsc, p: Permutation | None = None) -> FillReport:
    """Exact nnz(L) of P A P^T incl. diagonal (reference ordering.py:239-263)."""
    cp, ri = _csc(m)
    out = np.zeros(1, dtype=np.int64)
    f = None if p is None else i64arr(p.forward)
    check("tc_symbolic_fill_count", lib.tc_symbolic_fill_count(
        m.n, ptr(cp, i64p), ptr(ri, i32p), ptr(f, i64p), ptr(out, i64p)))
    return FillReport(nnz_original=m.nnz, nnz_factor=int(out[0]))


def factor_column_counts(m: SymmetricCsc, p: Permutation | None = None) -> np.ndarray:
    """nnz per column of L (incl. diagonal) of P A P^T (C++, etree row subtrees)."""
    cp, ri = _csc(m)
    out = np.empty(m.n, dtype=np.int64)
    f = None if p is None else i64arr(p.forward)
    check("tc_factor_column_counts", lib.tc_factor_column_counts(
        m.n, ptr(cp, i64p), ptr(ri, i32p), ptr(f, i64p), ptr(out, i64p)))
    return out


def select_ordering(m: SymmetricCsc, candidates) -> Permutation:
    """Identity unless a candidate has a strictly smaller factor; earlier
    candidates win ties (reference ordering.py:266-275).

    ``candidates`` may also hold zero-argument callables producing a
    Permutation: they are evaluated in order only while a strictly smaller
    factor is still possible.  nnz(L) of any symmetric permutation is at least
    nnz(lower A) (L's pattern contains PAP^T's), so when the identity has zero
    fill no candidate can win and none is computed -- the result is the one
    the reference's eager evaluation returns (e.g. BASELINE C1/C4, survey §8(a)
    row 8), without an RCM of a 2.5e9-entry pattern."""
    best = Permutation.identity(m.n)
    # parallel perfect-elimination test first: with zero fill the identity's
    # nnz(L) is nnz(lower A) without the sequential elimination-tree pass
    cp, ri = _csc(m)
    perfect, offd = np.zeros(1, dtype=np.int32), np.zeros(1, dtype=np.int64)
    check("tc_zero_fill", lib.tc_zero_fill(m.n, ptr(cp, i64p), ptr(ri, i32p), ptr(perfect, i32p), ptr(offd, i64p)))
    best_nnz = int(offd[0]) + m.n if perfect[0] else symbolic_fill_count(m, None).nnz_factor
    for cand in candidates:
        if best_nnz <= m.nnz:
            break
        if callable(cand):
            cand = cand()
        c = symbolic_fill_count(m, cand).nnz_factor
        if c < best_nnz:
            best, best_nnz = cand, c
    return best
