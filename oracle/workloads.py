"""Oracle-side synthetic inputs and bounded op-stream samples (TEST / BENCH
INFRASTRUCTURE ONLY — never imported by ``paper_2501_02483_b200``).

Everything here is numpy/scipy restated from SURVEY.md Appendix A, so the
reference CPU arm of ``bench.py`` never touches the product package or its
shared library:

* ``c1()``, ``c4_columns()`` — reference ``generate_arrowhead``
  (matcore.py:269-317): values ``default_rng(seed).uniform(-1, 1, nnz)`` in
  CSC order, diagonal = 1 + row-sum + column-sum of |off-diagonal| (bincount
  order).  ``c4_columns`` draws only the leading ``ncols`` columns: the PCG64
  stream of a prefix is the prefix of the stream, and every row-sum of a head
  row ``i < ncols`` only involves columns ``<= i``, so the prefix is
  bit-identical to the same columns of the full 2.5e9-entry matrix.
* ``c2()`` — App. A2 piecewise variable band.
* ``InlaFamily`` — App. A3 Q(theta) on one pattern (C3 / C5).
* ``prefix_problem`` / ``prefix_stream`` — the left-looking op stream
  (reference symbolic.py:126-164 + the SPEC.md:412-448 op compiler) of the
  first K tile columns, on a compact renumbering of the tile rows those
  columns touch: the ops of a column prefix only read and write tiles of that
  prefix, so the prefix is a self-contained, exactly-scaled sample of the full
  factorisation.
* ``arrowhead_tile_flops`` — closed-form tile-flop count of the zero-fill
  band + arrow pattern (N_SYRK = N_TRSM = sum |R_n|, N_GEMM = sum C(|R_n|, 2)).
"""

from __future__ import annotations

import math

import numpy as np

from . import core as O

__all__ = ["WORKLOAD_DESC", "c1", "c2", "c3", "c4_columns", "InlaFamily", "c5_thetas",
           "arrowhead_tile_rows", "arrowhead_tile_flops", "tile_flops_of_tasks", "prefix_problem"]

WORKLOAD_DESC = {
    "c1": "arrowhead n=10,000 b=200 t=50 (BASELINE config 1)",
    "c2": "variable-band arrowhead n=100,000 max band 1,000 t=200 (BASELINE config 2)",
    "c3": "INLA 2000x100+10 (n=200,010) kappa=.5 rho=.9 tau=1e-3 (BASELINE config 3)",
    "c4": "arrowhead n=1,000,000 b=2000 t=500 (BASELINE config 4)",
    "c5": "batch of 64 INLA factorizations (C3 pattern, theta on a 4x4x4 grid) (BASELINE config 5)",
}
C4_SPEC = (1_000_000, 2000, 500)


def _diag_rule(n, cp, ri, vals, cols=None):
    """diag = 1 + bincount(row, |v|) + bincount(col, |v|) (matcore.py:309-316)."""
    if cols is None:
        cols = np.repeat(np.arange(cp.size - 1, dtype=np.int64), np.diff(cp))
    mag = np.abs(vals)
    mag[cp[:-1]] = 0.0
    rs = np.bincount(ri, weights=mag, minlength=n)
    rs = rs + np.bincount(cols, weights=mag, minlength=n)
    vals[cp[:-1]] = rs[: cp.size - 1] + 1.0
    return vals


def _band_arrow(n, t, band, seed=0, ncols=None):
    """Head column j: rows j..j+band[j] then the t arrow rows; dense tail
    (reference generate_arrowhead layout, matcore.py:283-306)."""
    nh = n - t
    ncols = n if ncols is None else ncols
    lens = np.empty(ncols, dtype=np.int64)
    hc = min(ncols, nh)
    lens[:hc] = 1 + band[:hc] + t
    if ncols > nh:
        lens[nh:] = n - np.arange(nh, ncols, dtype=np.int64)
    cp = np.zeros(ncols + 1, dtype=np.int64)
    cp[1:] = np.cumsum(lens)
    nnz = int(cp[-1])
    cols = np.repeat(np.arange(ncols, dtype=np.int64), lens)
    pos = np.arange(nnz, dtype=np.int64) - cp[cols]
    rows = np.empty(nnz, dtype=np.int64)
    head = cols < nh
    bl = np.zeros(ncols, dtype=np.int64)
    bl[:hc] = band[:hc]
    inband = head & (pos <= bl[cols])
    rows[inband] = cols[inband] + pos[inband]
    arrow = head & ~inband
    rows[arrow] = nh + (pos[arrow] - bl[cols[arrow]] - 1)
    tail = ~head
    rows[tail] = cols[tail] + pos[tail]
    ri = rows.astype(np.int32)
    vals = np.random.default_rng(seed).uniform(-1.0, 1.0, size=nnz)
    return cp, ri, _diag_rule(n, cp, ri, vals, cols)


def c1():
    """(n, col_ptr, row_idx, values) of BASELINE config 1 (App. A1)."""
    n, b, t = 10_000, 200, 50
    band = np.minimum(b, (n - t) - 1 - np.arange(n - t, dtype=np.int64))
    return (n,) + _band_arrow(n, t, band, seed=0)


def c2(n=100_000, t=200, seg_len=5000, max_band=1000, min_band=100, seed=0, seg_seed=12345):
    """BASELINE config 2 (App. A2)."""
    nh = n - t
    seg = np.random.default_rng(seg_seed).integers(min_band, max_band + 1, size=math.ceil(nh / seg_len))
    seg[0] = max_band
    j = np.arange(nh, dtype=np.int64)
    band = np.minimum(seg[j // seg_len], nh - 1 - j)
    return (n,) + _band_arrow(n, t, band, seed=seed)


def c4_columns(ncols, n=C4_SPEC[0], b=C4_SPEC[1], t=C4_SPEC[2], seed=0):
    """The leading ``ncols`` (< n - t) columns of BASELINE config 4, bit-identical
    to those columns of the full generated matrix (module docstring)."""
    nh = n - t
    assert 0 < ncols <= nh
    band = np.minimum(b, nh - 1 - np.arange(ncols, dtype=np.int64))
    cp, ri, vals = _band_arrow(n, t, band, seed=seed, ncols=ncols)
    return n, cp, ri, vals


def c4_nnz(n=C4_SPEC[0], b=C4_SPEC[1], t=C4_SPEC[2]):
    return O.arrowhead_nnz(n, b, t)


class InlaFamily:
    """Q(theta) = [[Qt(rho) (x) Qs(kappa) + I, X], [X^T, X^T X + tau I]] on a
    40 x 50 grid, 100 time steps, 10 fixed effects (App. A3), as a linear
    combination of fixed basis value arrays on one union pattern."""

    def __init__(self, nx=40, ny=50, nsteps=100, nfix=10, seed=0):
        import scipy.sparse as sp

        def tri(k, lo, d, hi):
            return sp.diags([np.full(k - 1, lo), np.full(k, d), np.full(k - 1, hi)], [-1, 0, 1], format="csr")

        ns = nx * ny
        L = (sp.kron(sp.identity(ny), tri(nx, -1.0, 2.0, -1.0)) + sp.kron(tri(ny, -1.0, 2.0, -1.0),
                                                                          sp.identity(nx))).tocsr()
        space = [sp.identity(ns, format="csr"), L, (L @ L).tocsr()]
        d1 = np.ones(nsteps)
        d1[0] = d1[-1] = 0.0
        time_b = [sp.diags(np.ones(nsteps), 0), sp.diags(d1, 0),
                  sp.diags([np.ones(nsteps - 1), np.ones(nsteps - 1)], [-1, 1])]
        nl = ns * nsteps
        self.n = nl + nfix
        X = np.random.default_rng(seed).standard_normal((nl, nfix)) / math.sqrt(nl)
        XtX = X.T @ X
        blocks = [sp.kron(tb, sb, format="csr") for tb in time_b for sb in space]
        big = sum(abs(b) for b in blocks) + sp.identity(nl)
        full = sp.bmat([[big, sp.csr_matrix(np.ones((nl, nfix)))],
                        [sp.csr_matrix(np.ones((nfix, nl))), sp.csr_matrix(np.ones((nfix, nfix)))]])
        low = sp.tril(full, format="csc")
        low.sort_indices()
        self.col_ptr = low.indptr.astype(np.int64)
        self.row_idx = low.indices.astype(np.int32)
        self._key = np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.col_ptr)) * self.n \
            + self.row_idx.astype(np.int64)
        nnz = self.row_idx.size

        def on_pattern(mat):
            m = mat.tocoo()
            r, c = m.row.astype(np.int64), m.col.astype(np.int64)
            keep = r >= c
            v = np.zeros(nnz)
            np.add.at(v, self._locate(r[keep], c[keep]), m.data[keep])
            return v

        self.basis = {(i, j): on_pattern(blocks[3 * i + j]) for i in range(3) for j in range(3)}
        self.v_ident = on_pattern(sp.identity(nl))
        self.v_x = np.zeros(nnz)
        self.v_x[self._locate(np.repeat(np.arange(nl, self.n), nl), np.tile(np.arange(nl), nfix))] = X.T.ravel()
        fr, fc = np.tril_indices(nfix)
        self.v_xtx = np.zeros(nnz)
        self.v_xtx[self._locate(fr + nl, fc + nl)] = XtX[fr, fc]
        self.v_tau = np.zeros(nnz)
        self.v_tau[self._locate(np.arange(nl, self.n), np.arange(nl, self.n))] = 1.0

    def _locate(self, r, c):
        key = c * self.n + r
        pos = np.searchsorted(self._key, key)
        assert np.all(self._key[pos] == key)
        return pos

    def values(self, kappa, rho, tau):
        k2 = kappa * kappa
        cs = [k2 * k2, 2.0 * k2, 1.0]
        ct = [1.0, rho * rho, -rho]
        s = 1.0 / (1.0 - rho * rho)
        v = self.v_ident + self.v_x + self.v_xtx + tau * self.v_tau
        for i in range(3):
            for j in range(3):
                v = v + (s * ct[i] * cs[j]) * self.basis[(i, j)]
        return v


def c3(family=None):
    f = family or InlaFamily()
    return f.n, f.col_ptr, f.row_idx, f.values(0.5, 0.9, 1e-3)


def c5_thetas():
    return [(k, r, t) for k in (0.3, 0.5, 0.7, 0.9) for r in (0.5, 0.7, 0.9, 0.95)
            for t in (1e-4, 1e-3, 1e-2, 1e-1)]


# --------------------------------------------------------------------------
# tile flops and bounded prefix samples
# --------------------------------------------------------------------------

def tile_flops_of_tasks(ty, nt):
    """nt^3 (N_POTRF/3 + N_TRSM + N_SYRK + 2 N_GEMM) (survey §8 notation)."""
    c = np.bincount(np.asarray(ty, dtype=np.int64), minlength=7)
    return float(nt) ** 3 * (c[O.POTRF] / 3.0 + c[O.TRSM] + c[O.SYRK] + 2.0 * c[O.GEMM])


def arrowhead_tile_rows(n, b, t, nt, k):
    """Off-diagonal tile rows R_k of tile column k of the (zero-fill) band +
    arrow pattern: band tiles below the diagonal plus the arrow tiles."""
    nh = n - t
    T = -(-n // nt)
    c_lo, c_hi = k * nt, min(n, (k + 1) * nt) - 1
    rows = set()
    if c_lo < nh:
        last_band_row = min(min(c_hi, nh - 1) + b, nh - 1)
        rows.update(range(k + 1, last_band_row // nt + 1))
        rows.update(range(max(k + 1, nh // nt), T))
    else:
        rows.update(range(k + 1, T))
    return sorted(rows)


def arrowhead_tile_flops(n, b, t, nt):
    """Closed-form tile flops of the band + arrow pattern at identity ordering
    (zero fill, survey §8(a) row 8): N_SYRK = N_TRSM = sum_k |R_k|,
    N_GEMM = sum_k C(|R_k|, 2), N_POTRF = T."""
    T = -(-n // nt)
    s = 0
    g = 0
    for k in range(T):
        r = len(arrowhead_tile_rows(n, b, t, nt, k))
        s += r
        g += r * (r - 1) // 2
    return float(nt) ** 3 * (T / 3.0 + 2.0 * s + 2.0 * g), T + s


def prefix_problem(n, cp, ri, vals, nt, K, with_storage=True):
    """Bounded sample of one factorisation: the op stream of the first K tile
    columns of the matrix given by its leading columns (cp/ri/vals cover at
    least min(n, K*nt) columns), on a compact renumbering of the tile rows.

    Returns dict(op, dst, src1, src2, storage, flops, ops, slots, columns,
    grow, gcol): grow/gcol are the global (tile row, tile column) of every
    compact slot, so the sample's factor can be compared tile by tile with a
    factor of the whole matrix."""
    ncols = min(n, K * nt, cp.size - 1)
    cp = cp[: ncols + 1]
    nnz = int(cp[-1])
    ri = ri[:nnz]
    vals = vals[:nnz]
    cols = np.repeat(np.arange(ncols, dtype=np.int64), np.diff(cp))
    tr = ri.astype(np.int64) // nt
    tc = cols // nt
    Kc = int(-(-ncols // nt))
    used = np.union1d(np.unique(tr), np.arange(Kc, dtype=np.int64))
    comp = {int(g): i for i, g in enumerate(used)}
    cmap = np.searchsorted(used, tr)
    Tp = used.size
    # compact square problem: tile (cmap[r], c) for c < Kc
    keys = np.unique(cmap * Tp + tc)
    frows, fcols = keys // Tp, keys % Tp
    n_c = Tp * nt
    fr, fc, fsm, _ = O.tile_symbolic(n_c, nt, frows, fcols)
    tasks = O.task_stream(Tp, fsm)
    keep = tasks["k"] < Kc
    tasks = {kk: v[keep] for kk, v in tasks.items()}
    op, dst, s1, s2, _ = O.compile_ops(tasks, fsm, fr.size)
    st = None
    if with_storage:
        st = np.zeros((fr.size, nt, nt))
        flat = st.reshape(-1)
        slot = fsm[cmap, tc].astype(np.int64)
        flat[slot * nt * nt + (cols % nt) * nt + ri.astype(np.int64) % nt] = vals
        if ncols == n and n % nt:
            last = fsm[comp[int((n - 1) // nt)], Kc - 1]
            for loc in range(n % nt, nt):
                st[last, loc, loc] = 1.0
    return {"op": op, "dst": dst, "src1": s1, "src2": s2, "storage": st,
            "flops": tile_flops_of_tasks(tasks["type"], nt), "ops": int(op.size), "slots": int(fr.size),
            "columns": Kc, "grow": used[fr].astype(np.int64), "gcol": used[fc].astype(np.int64)}
