"""Oracle restatement (TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py).

Plain numpy for integer/structure work, numba-jitted scalar loops plus BLAS
(``np.dot``) for the FP64 tile numerics, i.e. the same arithmetic engine the
reference's default backend uses, so the oracle doubles as the CPU baseline.

Conventions (reference ctsf.py:87-105): tile storage is a C-order float64
array ``st[S, nt, nt]`` whose slot ``s`` holds element (i, j) of its tile at
``st[s, j, i]`` (column-major tile); ``st[s].T`` is the natural view.
"""

from __future__ import annotations

import heapq
import math

import numpy as np
from numba import njit

# op / task codes: reference symbolic.py:19-21, _backend_numba.py:13
POTRF, SYRK, TRSM, GEMM, GEADD, ZERO = 1, 2, 3, 4, 5, 6

__all__ = [
    "POTRF", "SYRK", "TRSM", "GEMM", "GEADD", "ZERO",
    "arrowhead", "arrowhead_nnz", "canonical", "structure", "permute", "tile_grid_of",
    "rcm_forward", "nd_forward", "min_degree_forward", "etree_count",
    "fill_count", "choose_ordering", "tile_grid", "tile_symbolic",
    "task_stream", "tree_plan", "combine_steps", "compile_ops", "pack",
    "dag_levels", "potrf_t", "trsm_t", "syrk_t", "gemm_t", "geadd_t",
    "run_ops", "replay_residual", "logdet", "tile_solve", "dense_of",
]


# --------------------------------------------------------------------------
# matrices (reference matcore.py)
# --------------------------------------------------------------------------

def arrowhead_nnz(n, b, t, block_diagonal=False):
    """Closed-form stored count; reference matcore.py:249-260."""
    nh = n - t
    if block_diagonal:
        q, r = divmod(nh, b)
        band = q * b * (b - 1) // 2 + r * (r - 1) // 2
    else:
        w = min(b, nh - 1)
        band = w * (nh - w) + w * (w - 1) // 2
    return n + band + t * (nh + n - 1) // 2


def arrowhead(n, b, t, block_diagonal=False, seed=0):
    """(col_ptr, row_idx, values) of the generated arrowhead; reference
    matcore.py:269-317 (same PCG64 draw order, same bincount row sums)."""
    nh = n - t
    j = np.arange(nh, dtype=np.int64)
    if block_diagonal:
        blen = np.minimum((j // b + 1) * b, nh) - j - 1
    else:
        blen = np.minimum(b, nh - 1 - j)
    lens = np.empty(n, dtype=np.int64)
    lens[:nh] = 1 + blen + t
    lens[nh:] = n - np.arange(nh, n, dtype=np.int64)
    cp = np.zeros(n + 1, dtype=np.int64)
    cp[1:] = np.cumsum(lens)
    nnz = int(cp[-1])
    rows = np.empty(nnz, dtype=np.int64)
    col_of = np.empty(nnz, dtype=np.int64)
    for c in range(n):  # per-column fill, clarity over speed
        lo = int(cp[c])
        if c < nh:
            nb = int(blen[c])
            rows[lo:lo + 1 + nb] = np.arange(c, c + 1 + nb)
            rows[lo + 1 + nb:cp[c + 1]] = np.arange(nh, n)
        else:
            rows[lo:cp[c + 1]] = np.arange(c, n)
        col_of[lo:cp[c + 1]] = c
    ridx = rows.astype(np.int32)
    vals = np.random.default_rng(seed).uniform(-1.0, 1.0, size=nnz)
    mag = np.abs(vals)
    mag[cp[:-1]] = 0.0
    rs = np.bincount(ridx, weights=mag, minlength=n)
    rs = rs + np.bincount(col_of, weights=mag, minlength=n)
    vals[cp[:-1]] = rs + 1.0
    return cp, ridx, vals


def canonical(n, rows, cols, vals, sum_duplicates=True):
    """Coordinates -> canonical lower CSC; reference matcore.py:89-133.
    Returns (col_ptr, row_idx, values) or raises ValueError(msg)."""
    r = np.asarray(rows, dtype=np.int64)
    c = np.asarray(cols, dtype=np.int64)
    v = np.asarray(vals, dtype=np.float64)
    lo_r = np.maximum(r, c)
    lo_c = np.minimum(r, c)
    perm = np.lexsort((lo_r, lo_c))
    lo_r, lo_c, v = lo_r[perm], lo_c[perm], v[perm]
    if lo_r.size:
        first = np.ones(lo_r.size, dtype=bool)
        first[1:] = (lo_r[1:] != lo_r[:-1]) | (lo_c[1:] != lo_c[:-1])
        if not first.all():
            if not sum_duplicates:
                raise ValueError("duplicate entries present")
            v = np.add.reduceat(v, np.flatnonzero(first))
            lo_r, lo_c = lo_r[first], lo_c[first]
    cp = np.zeros(n + 1, dtype=np.int64)
    cp[1:] = np.cumsum(np.bincount(lo_c, minlength=n))
    return cp, lo_r.astype(np.int32), v


def structure(n, cp, ri, thr=0.5):
    """(bandwidth, thickness, density%); reference matcore.py:320-348."""
    cnt = np.bincount(ri, minlength=n).astype(np.int64) + np.diff(cp) - 1
    t = 0
    while t < n and cnt[n - 1 - t] >= thr * n:
        t += 1
    cols = np.repeat(np.arange(n), np.diff(cp))
    keep = ri < n - t
    bw = int((ri[keep].astype(np.int64) - cols[keep]).max(initial=0))
    dens = 100.0 * (2 * int(cp[-1]) - n) / (n * n)
    return bw, t, dens


def permute(n, cp, ri, vals, fwd):
    """B[p(i), p(j)] = A[i, j]; reference matcore.py:351-366."""
    cols = np.repeat(np.arange(n, dtype=np.int64), np.diff(cp))
    return canonical(n, fwd[ri.astype(np.int64)], fwd[cols], vals, sum_duplicates=False)


def dense_of(n, cp, ri, vals):
    a = np.zeros((n, n))
    cols = np.repeat(np.arange(n), np.diff(cp))
    a[ri, cols] = vals
    a[cols, ri] = vals
    return a


# --------------------------------------------------------------------------
# orderings (reference ordering.py)
# --------------------------------------------------------------------------

def _head_graph(n, cp, ri, limit):
    """Adjacency lists of the head subgraph; reference ordering.py:83-97."""
    cols = np.repeat(np.arange(n, dtype=np.int64), np.diff(cp))
    rr = ri.astype(np.int64)
    m = (rr != cols) & (rr < limit)
    a = np.concatenate([rr[m], cols[m]])
    b = np.concatenate([cols[m], rr[m]])
    o = np.lexsort((b, a))
    a, b = a[o], b[o]
    ptr = np.zeros(limit + 1, dtype=np.int64)
    ptr[1:] = np.cumsum(np.bincount(a, minlength=limit))
    return [b[ptr[v]:ptr[v + 1]].tolist() for v in range(limit)]


def _levels(adj, root):
    """BFS levels, each sorted ascending; reference ordering.py:100-115."""
    seen = {root}
    out = [[root]]
    while True:
        frontier = []
        for v in out[-1]:
            for w in adj[v]:
                if w not in seen:
                    seen.add(w)
                    frontier.append(w)
        if not frontier:
            return out
        frontier.sort()
        out.append(frontier)


def _peripheral(adj, start, deg):
    """George-Liu root search; reference ordering.py:118-131."""
    root = start
    lv = _levels(adj, root)
    while True:
        cand = min(lv[-1], key=lambda v: (deg[v], v))
        if cand == root:
            return root
        lv2 = _levels(adj, cand)
        if len(lv2) <= len(lv):
            return cand
        root, lv = cand, lv2


def rcm_forward(n, cp, ri, pinned_tail=0):
    """Partial RCM forward map; reference ordering.py:134-170."""
    nh = n - pinned_tail
    adj = _head_graph(n, cp, ri, nh)
    deg = [len(a) for a in adj]
    seen = [False] * nh
    order = []
    for s in range(nh):
        if seen[s]:
            continue
        r = _peripheral(adj, s, deg)
        seen[r] = True
        q = [r]
        h = 0
        while h < len(q):
            v = q[h]
            h += 1
            order.append(v)
            kids = sorted((w for w in adj[v] if not seen[w]), key=lambda w: (deg[w], w))
            for w in kids:
                seen[w] = True
                q.append(w)
    fwd = np.arange(n, dtype=np.int64)
    fwd[np.asarray(order[::-1], dtype=np.int64)] = np.arange(nh, dtype=np.int64)
    return fwd


def nd_forward(n, bw, t, max_levels=8):
    """Adaptable nested dissection; reference ordering.py:209-236."""
    groups = []

    def split(lo, hi, lvl):
        sz = hi - lo
        if bw == 0 or lvl >= max_levels or sz <= 4 * bw:
            groups.append((lo, hi))
            return
        mid = lo + sz // 2
        split(lo, mid, lvl + 1)
        split(mid + bw, hi, lvl + 1)
        groups.append((mid, mid + bw))

    split(0, n - t, 0)
    groups.append((n - t, n))
    old = np.concatenate([np.arange(a, b, dtype=np.int64) for a, b in groups])
    fwd = np.empty(n, dtype=np.int64)
    fwd[old] = np.arange(n, dtype=np.int64)
    return fwd


def min_degree_forward(n, cp, ri):
    """Exact greedy minimum degree; reference ordering.py:173-206."""
    adj = [set(a) for a in _head_graph(n, cp, ri, n)]
    alive = [True] * n
    pq = [(len(adj[v]), v) for v in range(n)]
    heapq.heapify(pq)
    fwd = np.empty(n, dtype=np.int64)
    for step in range(n):
        while True:
            d, v = heapq.heappop(pq)
            if alive[v] and d == len(adj[v]):
                break
        alive[v] = False
        fwd[v] = step
        nb = adj[v]
        for w in nb:
            adj[w].discard(v)
        nbs = sorted(nb)
        for i, a in enumerate(nbs):
            for b in nbs[i + 1:]:
                if b not in adj[a]:
                    adj[a].add(b)
                    adj[b].add(a)
        for w in nbs:
            heapq.heappush(pq, (len(adj[w]), w))
        adj[v] = set()
    return fwd


@njit(cache=True)
def etree_count(n, ptr, cols):
    """Strict-lower nnz(L) via Liu's etree + row subtrees; reference
    _backend_numba.py:188-215."""
    par = np.full(n, -1, np.int64)
    anc = np.full(n, -1, np.int64)
    for i in range(n):
        for p in range(ptr[i], ptr[i + 1]):
            r = cols[p]
            while anc[r] != -1 and anc[r] != i:
                nx = anc[r]
                anc[r] = i
                r = nx
            if anc[r] == -1:
                anc[r] = i
                par[r] = i
    flag = np.full(n, -1, np.int64)
    total = 0
    for i in range(n):
        flag[i] = i
        for p in range(ptr[i], ptr[i + 1]):
            r = cols[p]
            while flag[r] != i:
                flag[r] = i
                total += 1
                r = par[r]
    return total


def fill_count(n, cp, ri, fwd=None):
    """nnz(L) incl. diagonal; reference ordering.py:239-263."""
    if fwd is None:
        fwd = np.arange(n, dtype=np.int64)
    cols = np.repeat(np.arange(n, dtype=np.int64), np.diff(cp))
    rr = ri.astype(np.int64)
    off = rr != cols
    pi, pj = fwd[rr[off]], fwd[cols[off]]
    hi, lo = np.maximum(pi, pj), np.minimum(pi, pj)
    o = np.argsort(hi, kind="stable")
    hi, lo = hi[o], lo[o]
    ptr = np.zeros(n + 1, dtype=np.int64)
    ptr[1:] = np.cumsum(np.bincount(hi, minlength=n))
    return int(etree_count(n, ptr, lo.astype(np.int64))) + n


def choose_ordering(n, cp, ri, candidates):
    """Identity unless a candidate is strictly smaller (earlier wins ties);
    reference ordering.py:266-275.  Returns (forward, index) with index -1 for
    identity."""
    best = np.arange(n, dtype=np.int64)
    best_c = fill_count(n, cp, ri, best)
    which = -1
    for i, f in enumerate(candidates):
        c = fill_count(n, cp, ri, f)
        if c < best_c:
            best, best_c, which = f, c, i
    return best, which


# --------------------------------------------------------------------------
# tiles, symbolic, task stream (reference ctsf.py, symbolic.py)
# --------------------------------------------------------------------------

def tile_grid(n, nt, trows, tcols):
    """Occupied lower tiles + all diagonals in (col,row) slot order;
    reference ctsf.py:57-75.  Returns (tile_rows, tile_cols, slot_map)."""
    T = -(-n // nt)
    tr = np.asarray(trows, dtype=np.int64)
    tc = np.asarray(tcols, dtype=np.int64)
    occ = np.zeros((T, T), dtype=bool)
    occ[np.maximum(tr, tc), np.minimum(tr, tc)] = True
    occ[np.arange(T), np.arange(T)] = True
    # slot order = column-major scan of the lower triangle
    cc, rr = np.nonzero(occ.T)
    sm = np.full((T, T), -1, dtype=np.int32)
    sm[rr, cc] = np.arange(rr.size, dtype=np.int32)
    return rr.astype(np.int32), cc.astype(np.int32), sm


def tile_grid_of(n, nt, cp, ri):
    """reference ctsf.py:78-84."""
    cols = np.repeat(np.arange(n, dtype=np.int64), np.diff(cp))
    return tile_grid(n, nt, ri.astype(np.int64) // nt, cols // nt)


def tile_symbolic(n, nt, trows, tcols):
    """Tile elimination game + accumulation counts; reference
    symbolic.py:98-123.  Returns (f_rows, f_cols, f_slot_map, accum)."""
    T = -(-n // nt)
    f = np.zeros((T, T), dtype=bool)
    f[trows, tcols] = True
    for k in range(T):
        below = k + 1 + np.flatnonzero(f[k + 1:, k])
        if below.size > 1:
            f[np.ix_(below, below)] = True
    low = np.tril(f)
    r, c = np.nonzero(low)
    fr, fc, fsm = tile_grid(n, nt, r, c)
    strict = np.tril(low, -1)
    acc = np.zeros(fr.size, dtype=np.int64)
    for k in range(T):
        rowk = strict[k, :k]
        acc[fsm[k, k]] = int(rowk.sum())
        ms = k + np.flatnonzero(strict[k:, k])
        for m in ms:
            acc[fsm[m, k]] = int(np.count_nonzero(strict[m, :k] & rowk))
    return fr, fc, fsm, acc


def task_stream(T, fsm):
    """Left-looking task stream; reference symbolic.py:126-164.
    Returns dict of arrays type(int8), m, k, n, target (int32)."""
    L = fsm >= 0
    strict = np.tril(L, -1)
    ty, mm, kk, nn = [], [], [], []
    for k in range(T):
        for n in np.flatnonzero(strict[k, :k]):
            ty.append(SYRK); mm.append(k); kk.append(k); nn.append(int(n))
        ty.append(POTRF); mm.append(k); kk.append(k); nn.append(0)
        for m in k + 1 + np.flatnonzero(strict[k + 1:, k]):
            for n in np.flatnonzero(strict[m, :k] & strict[k, :k]):
                ty.append(GEMM); mm.append(int(m)); kk.append(k); nn.append(int(n))
            ty.append(TRSM); mm.append(int(m)); kk.append(k); nn.append(0)
    m = np.asarray(mm, dtype=np.int32)
    k = np.asarray(kk, dtype=np.int32)
    return {"type": np.asarray(ty, dtype=np.int8), "m": m, "k": k,
            "n": np.asarray(nn, dtype=np.int32),
            "target": fsm[m, k].astype(np.int32)}


def combine_steps(w):
    """Balanced pairwise GEADD tree; reference symbolic.py:241-250."""
    out = []
    s = 1
    while s < w:
        out.extend((a, a + s) for a in range(0, w, 2 * s) if a + s < w)
        s *= 2
    return out


def tree_plan(accum, workers):
    """slot -> list of [start, end) chain ranges; reference
    symbolic.py:253-269."""
    plan = {}
    for s in np.flatnonzero(np.asarray(accum) >= 2 * workers):
        c = int(accum[s])
        q, r = divmod(c, workers)
        sizes = [q + 1] * r + [q] * (workers - r)
        e = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        plan[int(s)] = [(int(e[i]), int(e[i + 1])) for i in range(workers)]
    return plan


def compile_ops(tasks, fsm, S, plan=None, workers=0):
    """Task stream -> (op_type, dst, src1, src2, n_scratch).

    Reconstruction of the reference's missing scheduler op compiler
    (survey §8(a) row 24): SYRK src1=slot(k,n); TRSM
    src1=slot(k,k); GEMM src1=slot(k,n), src2=slot(m,n).  Planned chains
    (SPEC.md:421-424, :443): ZERO each scratch, the chain ops in range w
    redirected to scratch w, the combine GEADDs, GEADD(target, scratch 0),
    then the finalising POTRF/TRSM.  Scratch slot ids are S + w.
    """
    ty, m, k, n, tgt = (tasks[x] for x in ("type", "m", "k", "n", "target"))
    P = ty.size
    s1 = np.full(P, -1, np.int64)
    s2 = np.full(P, -1, np.int64)
    isy = ty == SYRK
    s1[isy] = fsm[k[isy], n[isy]]
    itr = ty == TRSM
    s1[itr] = fsm[k[itr], k[itr]]
    ige = ty == GEMM
    s1[ige] = fsm[k[ige], n[ige]]
    s2[ige] = fsm[m[ige], n[ige]]
    dst = tgt.astype(np.int64)
    if not plan:
        return ty.astype(np.int8), dst, s1, s2, 0
    W = workers
    o_t, o_d, o_1, o_2 = [], [], [], []

    def emit(t, d, a, b):
        o_t.append(t); o_d.append(d); o_1.append(a); o_2.append(b)

    p = 0
    while p < P:
        q = p
        while q < P and dst[q] == dst[p]:
            q += 1
        slot = int(dst[p])
        if slot in plan:
            chain = list(range(p, q - 1))  # accumulation ops; op q-1 finalises
            for w in range(W):
                emit(ZERO, S + w, -1, -1)
            for w, (a, b) in enumerate(plan[slot]):
                for i in chain[a:b]:
                    emit(int(ty[i]), S + w, int(s1[i]), int(s2[i]))
            for a, b in combine_steps(W):
                emit(GEADD, S + a, S + b, -1)
            emit(GEADD, slot, S, -1)
            emit(int(ty[q - 1]), slot, int(s1[q - 1]), int(s2[q - 1]))
        else:
            for i in range(p, q):
                emit(int(ty[i]), int(dst[i]), int(s1[i]), int(s2[i]))
        p = q
    return (np.asarray(o_t, np.int8), np.asarray(o_d, np.int64),
            np.asarray(o_1, np.int64), np.asarray(o_2, np.int64), W)


def pack(n, nt, cp, ri, vals, fsm, S):
    """Scatter CSC values into tile storage + unit padding; reference
    ctsf.py:118-139."""
    st = np.zeros((S, nt, nt))
    flat = st.reshape(-1)
    cols = np.repeat(np.arange(n, dtype=np.int64), np.diff(cp))
    rr = ri.astype(np.int64)
    slot = fsm[rr // nt, cols // nt].astype(np.int64)
    assert slot.min(initial=0) >= 0
    flat[slot * nt * nt + (cols % nt) * nt + rr % nt] = vals
    T = -(-n // nt)
    for loc in range(n % nt or nt, nt):
        st[fsm[T - 1, T - 1], loc, loc] = 1.0
    return st


def dag_levels(T, fsm, tasks):
    """Unit-cost DAG layering -> (critical_path, max_width); reference
    symbolic.py:287-331."""
    ty, m, k, n, tgt = (tasks[x] for x in ("type", "m", "k", "n", "target"))
    P = ty.size
    last = {}
    for p in range(P):
        last[int(tgt[p])] = p
    lvl = np.zeros(P, dtype=np.int64)
    for p in range(P):
        deps = []
        if p and tgt[p] == tgt[p - 1]:
            deps.append(p - 1)
        if ty[p] == SYRK:
            deps.append(last[int(fsm[k[p], n[p]])])
        elif ty[p] == GEMM:
            deps += [last[int(fsm[k[p], n[p]])], last[int(fsm[m[p], n[p]])]]
        elif ty[p] == TRSM:
            deps.append(last[int(fsm[k[p], k[p]])])
        lvl[p] = max((lvl[d] + 1 for d in deps), default=0)
    if not P:
        return 0, 0
    return int(lvl.max()) + 1, int(np.bincount(lvl).max())


# --------------------------------------------------------------------------
# FP64 tile numerics (reference _backend_numba.py:16-185)
# --------------------------------------------------------------------------

@njit(cache=True, nogil=True)
def potrf_t(a):
    """Right-looking scalar Cholesky on the natural view; -1 or pivot index.
    reference _backend_numba.py:16-38 (``d <= 0`` predicate, NaN passes)."""
    nt = a.shape[0]
    for j in range(nt):
        piv = a[j, j]
        if piv <= 0.0:
            return j
        piv = math.sqrt(piv)
        a[j, j] = piv
        r = 1.0 / piv
        for i in range(j + 1, nt):
            a[i, j] *= r
        for c in range(j + 1, nt):
            f = a[c, j]
            if f != 0.0:
                for i in range(c, nt):
                    a[i, c] -= a[i, j] * f
    for c in range(1, nt):
        for i in range(c):
            a[i, c] = 0.0
    return -1


@njit(cache=True, nogil=True)
def trsm_t(l, x):
    """X L^T = B in place; -1 or zero-diagonal index.
    reference _backend_numba.py:41-59."""
    nt = l.shape[0]
    for c in range(nt):
        d = l[c, c]
        if d == 0.0:
            return c
        r = 1.0 / d
        for i in range(nt):
            x[i, c] *= r
        for j in range(c + 1, nt):
            f = l[j, c]
            if f != 0.0:
                for i in range(nt):
                    x[i, j] -= x[i, c] * f
    return -1


@njit(cache=True, nogil=True)
def syrk_t(a, c):
    """c -= a a^T (full tile); reference _backend_numba.py:62-69."""
    prod = np.dot(a, a.T)
    nt = a.shape[0]
    for j in range(nt):
        for i in range(nt):
            c[i, j] -= prod[j, i]


@njit(cache=True, nogil=True)
def gemm_t(a, b, c):
    """c -= b a^T; reference _backend_numba.py:72-79."""
    prod = np.dot(a, b.T)
    nt = a.shape[0]
    for j in range(nt):
        for i in range(nt):
            c[i, j] -= prod[j, i]


@njit(cache=True, nogil=True)
def geadd_t(t, c):
    """c += t; reference _backend_numba.py:82-88."""
    nt = t.shape[0]
    for j in range(nt):
        for i in range(nt):
            c[i, j] += t[i, j]


@njit(cache=True, nogil=True)
def _view(st, sc, s):
    if s < st.shape[0]:
        return st[s].T
    return sc[s - st.shape[0]].T


@njit(cache=True, nogil=True)
def run_ops(st, sc, op, dst, s1, s2, start, stop):
    """Sequential op-stream executor; reference _backend_numba.py:98-133."""
    for p in range(start, stop):
        t = op[p]
        if t == GEMM:
            gemm_t(_view(st, sc, s1[p]), _view(st, sc, s2[p]), _view(st, sc, dst[p]))
        elif t == SYRK:
            syrk_t(_view(st, sc, s1[p]), _view(st, sc, dst[p]))
        elif t == TRSM:
            e = trsm_t(_view(st, sc, s1[p]), _view(st, sc, dst[p]))
            if e >= 0:
                return p, e
        elif t == POTRF:
            e = potrf_t(_view(st, sc, dst[p]))
            if e >= 0:
                return p, e
        elif t == GEADD:
            geadd_t(_view(st, sc, s1[p]), _view(st, sc, dst[p]))
        else:
            v = _view(st, sc, dst[p])
            v[:, :] = 0.0
    return stop, -1


@njit(cache=True, nogil=True)
def replay_residual(st, tpl, op, dst, s1, s2, is_diag):
    """sum ||(L L^T)_tile - A_tile||^2 with symmetric weights; reference
    _backend_numba.py:136-185 (sequential stream, no scratch)."""
    nt = st.shape[1]
    P = op.shape[0]
    acc = np.zeros((nt, nt))
    tot = 0.0
    cur = -1
    for p in range(P + 1):
        d = dst[p] if p < P else -2
        if d != cur:
            if cur >= 0:
                ref = tpl[cur].T
                for j in range(nt):
                    for i in range(nt):
                        if is_diag[cur]:
                            if i < j:
                                continue
                            w = 1.0 if i == j else 2.0
                        else:
                            w = 2.0
                        e = acc[i, j] - ref[i, j]
                        tot += w * e * e
            if p == P:
                break
            acc[:, :] = 0.0
            cur = d
        t = op[p]
        if t == POTRF:
            acc += np.dot(st[d].T, st[d])
        elif t == SYRK:
            acc += np.dot(st[s1[p]].T, st[s1[p]])
        elif t == TRSM:
            acc += np.dot(st[d].T, st[s1[p]])
        else:
            acc += np.dot(st[s2[p]].T, st[s1[p]])
    return tot


def logdet(st, fsm, n, nt):
    """2 sum log diag(L) over non-padding positions."""
    T = fsm.shape[0]
    tot = 0.0
    for k in range(T):
        d = np.diagonal(st[fsm[k, k]].T)
        live = min(nt, n - k * nt)
        tot += float(np.sum(np.log(d[:live])))
    return 2.0 * tot


def tile_solve(st, fsm, n, nt, b, fwd=None):
    """x = P^T L^-T L^-1 P b by tile forward/back substitution
    (permutation convention ordering.py:18-24)."""
    from scipy.linalg import solve_triangular
    T = fsm.shape[0]
    b = np.asarray(b, dtype=np.float64)
    if fwd is not None:
        inv = np.empty_like(fwd)
        inv[fwd] = np.arange(n)
        b = b[inv]
    y = np.zeros(T * nt)
    y[:n] = b
    L = fsm >= 0
    for k in range(T):
        yk = y[k * nt:(k + 1) * nt]
        for c in np.flatnonzero(L[k, :k]):
            yk -= st[fsm[k, c]].T @ y[c * nt:(c + 1) * nt]
        yk[:] = solve_triangular(st[fsm[k, k]].T, yk, lower=True)
    for k in range(T - 1, -1, -1):
        yk = y[k * nt:(k + 1) * nt]
        for r in k + 1 + np.flatnonzero(L[k + 1:, k]):
            yk -= st[fsm[r, k]] @ y[r * nt:(r + 1) * nt]
        yk[:] = solve_triangular(st[fsm[k, k]].T, yk, lower=True, trans="T")
    x = y[:n]
    if fwd is not None:
        x = x[fwd]
    return x.copy()
