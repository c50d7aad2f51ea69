"""Synthetic inputs of the BASELINE.json configurations (survey Appendix A).

C1/C4: the reference ``generate_arrowhead`` (matcore.py:269-317), bit-identical.
C2: piecewise variable-band arrowhead (App. A2), same value/diagonal rule.
C3/C5: INLA spatio-temporal precision Q(theta) = [[Qt(rho) (x) Qs(kappa) + I, X],
[X^T, X^T X + tau I]] on a 40 x 50 grid, 100 time steps, 10 fixed effects
(App. A3).  All C5 problems share one pattern; their values are a linear
combination of fixed basis value arrays (exact up to rounding of the
combination), so a 64-problem batch is generated in seconds.
"""

from __future__ import annotations

import math

import numpy as np

from ._lib import check, f64p, i32p, i64p, lib, ptr
from .matcore import ArrowheadSpec, SymmetricCsc, generate_arrowhead

__all__ = ["c1", "c2_variable_band", "c4", "InlaFamily", "c3", "c5_thetas"]


def c1() -> SymmetricCsc:
    """BASELINE config 1: n=10,000, b=200, t=50."""
    return generate_arrowhead(ArrowheadSpec(n=10_000, b=200, t=50, seed=0))


def c4() -> SymmetricCsc:
    """BASELINE config 4: n=1,000,000, b=2000, t=500 (2.5e9 stored entries)."""
    return generate_arrowhead(ArrowheadSpec(n=1_000_000, b=2000, t=500, seed=0))


def band_arrow(n: int, t: int, band: np.ndarray, seed: int = 0) -> SymmetricCsc:
    """Head column j: rows j..j+band[j] + the t arrow rows; dense tail.
    Values uniform(-1, 1) in CSC order, diagonal = 1 + |row| sum."""
    band = np.ascontiguousarray(band, dtype=np.int64)
    cp = np.empty(n + 1, dtype=np.int64)
    check("tc_band_arrow_pattern", lib.tc_band_arrow_pattern(n, t, ptr(band, i64p), ptr(cp, i64p), None))
    nnz = int(cp[-1])
    ri = np.empty(nnz, dtype=np.int32)
    check("tc_band_arrow_pattern", lib.tc_band_arrow_pattern(n, t, ptr(band, i64p), ptr(cp, i64p),
                                                             ptr(ri, i32p)))
    vals = np.random.default_rng(seed).uniform(-1.0, 1.0, size=nnz)
    check("tc_arrowhead_diag", lib.tc_arrowhead_diag(n, ptr(cp, i64p), ptr(ri, i32p), ptr(vals, f64p)))
    return SymmetricCsc(n, cp, ri, vals)


def c2_variable_band(n: int = 100_000, t: int = 200, seg_len: int = 5000, max_band: int = 1000,
                     min_band: int = 100, seed: int = 0, seg_seed: int = 12345) -> SymmetricCsc:
    """BASELINE config 2 (App. A2): band per 5,000-column segment from
    default_rng(12345).integers(100, 1001), first segment 1000."""
    nh = n - t
    seg = np.random.default_rng(seg_seed).integers(min_band, max_band + 1, size=math.ceil(nh / seg_len))
    seg[0] = max_band
    j = np.arange(nh, dtype=np.int64)
    band = np.minimum(seg[j // seg_len], nh - 1 - j)
    return band_arrow(n, t, band, seed=seed)


def _tridiag(k: int, lo: float, d, hi: float):
    import scipy.sparse as sp
    dd = np.full(k, d, dtype=np.float64) if np.isscalar(d) else np.asarray(d, dtype=np.float64)
    return sp.diags([np.full(k - 1, lo), dd, np.full(k - 1, hi)], [-1, 0, 1], format="csr")


class InlaFamily:
    """Q(theta) on one fixed pattern for theta = (kappa, rho, tau)."""

    def __init__(self, nx: int = 40, ny: int = 50, nsteps: int = 100, nfix: int = 10, seed: int = 0):
        import scipy.sparse as sp
        ns = nx * ny
        T1 = _tridiag(nx, -1.0, 2.0, -1.0)
        T2 = _tridiag(ny, -1.0, 2.0, -1.0)
        L = (sp.kron(sp.identity(ny), T1) + sp.kron(T2, sp.identity(nx))).tocsr()
        Is = sp.identity(ns, format="csr")
        space = [Is, L, (L @ L).tocsr()]            # Qs = k^4 I + 2 k^2 L + L^2
        d0 = np.ones(nsteps)
        d1 = np.ones(nsteps)
        d1[0] = d1[-1] = 0.0
        time_b = [sp.diags(d0, 0), sp.diags(d1, 0),
                  sp.diags([np.ones(nsteps - 1), np.ones(nsteps - 1)], [-1, 1])]  # Qt=(D0+r^2 D1-r E)/(1-r^2)
        nl = ns * nsteps
        self.n = nl + nfix
        X = np.random.default_rng(seed).standard_normal((nl, nfix)) / math.sqrt(nl)
        XtX = X.T @ X
        # union pattern: every kron(time_i, space_j) lower part, identity, X block, dense fixed block
        blocks = []
        for tb in time_b:
            for sb in space:
                blocks.append(sp.kron(tb, sb, format="csr"))
        big = sum(abs(b) for b in blocks) + sp.identity(nl)
        fullpat = sp.bmat([[big, sp.csr_matrix(np.ones((nl, nfix)))],
                           [sp.csr_matrix(np.ones((nfix, nl))), sp.csr_matrix(np.ones((nfix, nfix)))]])
        low = sp.tril(fullpat, format="csc")
        low.sort_indices()
        self.col_ptr = low.indptr.astype(np.int64)
        self.row_idx = low.indices.astype(np.int32)
        nnz = self.row_idx.size
        cols = np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.col_ptr))
        rows = self.row_idx.astype(np.int64)
        self._cols, self._rows = cols, rows

        def on_pattern(mat, off_r=0, off_c=0):
            m = mat.tocoo()
            v = np.zeros(nnz)
            r = m.row.astype(np.int64) + off_r
            c = m.col.astype(np.int64) + off_c
            keep = r >= c
            pos = self._locate(r[keep], c[keep])
            np.add.at(v, pos, m.data[keep])
            return v

        self.basis = {(i, j): on_pattern(blocks[3 * i + j]) for i in range(3) for j in range(3)}
        self.v_ident = on_pattern(sp.identity(nl))
        xr = np.repeat(np.arange(nl, self.n), nl)
        xc = np.tile(np.arange(nl), nfix)
        self.v_x = np.zeros(nnz)
        self.v_x[self._locate(xr, xc)] = X.T.ravel()
        fr, fc = np.tril_indices(nfix)
        self.v_xtx = np.zeros(nnz)
        self.v_xtx[self._locate(fr + nl, fc + nl)] = XtX[fr, fc]
        self.v_tau = np.zeros(nnz)
        self.v_tau[self._locate(np.arange(nl, self.n), np.arange(nl, self.n))] = 1.0

    def _locate(self, r, c):
        key = c * self.n + r
        allkey = self._cols * self.n + self._rows
        pos = np.searchsorted(allkey, key)
        assert np.all(allkey[pos] == key)
        return pos

    def values(self, kappa: float, rho: float, tau: float) -> np.ndarray:
        k2 = kappa * kappa
        cs = [k2 * k2, 2.0 * k2, 1.0]                       # space coefficients
        ct = [1.0, rho * rho, -rho]                         # time coefficients
        s = 1.0 / (1.0 - rho * rho)
        v = self.v_ident + self.v_x + self.v_xtx + tau * self.v_tau
        for i in range(3):
            for j in range(3):
                v = v + (s * ct[i] * cs[j]) * self.basis[(i, j)]
        return v

    def lincomb(self, kappa: float, rho: float, tau: float):
        """(coefficients, basis vectors) with values(theta) == the left-to-right
        sum of coef[i] * basis[i] (separately rounded products and sums; the
        unit coefficients are exact), for device-side assembly
        (tc_plan_pack_lincomb)."""
        k2 = kappa * kappa
        cs = [k2 * k2, 2.0 * k2, 1.0]
        ct = [1.0, rho * rho, -rho]
        s = 1.0 / (1.0 - rho * rho)
        coef = [1.0, 1.0, 1.0, tau] + [s * ct[i] * cs[j] for i in range(3) for j in range(3)]
        basis = [self.v_ident, self.v_x, self.v_xtx, self.v_tau] + [self.basis[(i, j)] for i in range(3)
                                                                      for j in range(3)]
        return coef, basis

    def matrix(self, kappa: float, rho: float, tau: float) -> SymmetricCsc:
        return SymmetricCsc(self.n, self.col_ptr, self.row_idx, self.values(kappa, rho, tau))


def c3(family: InlaFamily | None = None) -> SymmetricCsc:
    """BASELINE config 3: kappa=0.5, rho=0.9, tau=1e-3."""
    return (family or InlaFamily()).matrix(0.5, 0.9, 1e-3)


def c5_thetas():
    """The 64 (kappa, rho, tau) points of BASELINE config 5 (4 x 4 x 4 grid)."""
    return [(k, r, t) for k in (0.3, 0.5, 0.7, 0.9) for r in (0.5, 0.7, 0.9, 0.95)
            for t in (1e-4, 1e-3, 1e-2, 1e-1)]
