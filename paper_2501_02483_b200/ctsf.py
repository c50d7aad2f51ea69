"""Compressed tile storage (reference ctsf.py): occupied-tile grids in
(tile column, tile row) slot order and contiguous column-major tiles.

``TiledMatrix.storage`` is either a host numpy array or a CUDA torch tensor of
shape (S, nt, nt), C order, element (i, j) of slot s at ``storage[s, j, i]`` —
the same bytes the reference produces, so factors can be compared slot by
slot.  The dense ``slot_map`` is materialised lazily (it is T x T).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import check, i32p, i64p, lib, ptr
from .matcore import SymmetricCsc, from_coordinates

__all__ = ["TileGrid", "grid_from_tiles", "build_tile_grid", "TiledMatrix",
           "pack_into_grid", "pack_ctsf", "expand_to_grid", "unpack_to_csc"]


class _Sym:
    """Owner of a C ``tc_symbolic_t`` handle."""

    def __init__(self, handle: int):
        self.h = C.c_void_p(handle)

    def __del__(self):
        # at interpreter shutdown the module globals may already be gone
        if getattr(self, "h", None) and self.h.value and lib is not None:
            lib.tc_symbolic_destroy(self.h)
            self.h = C.c_void_p(0)

    def info(self):
        v = [np.zeros(1, dtype=np.int64) for _ in range(4)]
        check("tc_symbolic_info", lib.tc_symbolic_info(self.h, *(ptr(x, i64p) for x in v)))
        return tuple(int(x[0]) for x in v)  # T, S_in, S, P


def _sym_from_csc(m: SymmetricCsc, nt: int) -> _Sym:
    h = C.c_void_p()
    cp, ri = _lib.i64arr(m.col_ptr), _lib.i32arr(m.row_idx)
    check("tc_symbolic_from_csc", lib.tc_symbolic_from_csc(m.n, nt, ptr(cp, i64p), ptr(ri, i32p),
                                                           C.byref(h)))
    return _Sym(h.value)


def _sym_from_tiles(n: int, nt: int, rows, cols) -> _Sym:
    h = C.c_void_p()
    r, c = _lib.i64arr(rows), _lib.i64arr(cols)
    check("tc_symbolic_from_tiles", lib.tc_symbolic_from_tiles(n, nt, r.size, ptr(r, i64p),
                                                               ptr(c, i64p), C.byref(h)))
    return _Sym(h.value)


@dataclass(eq=False)
class TileGrid:
    """Occupied lower tiles (reference ctsf.py:21-54)."""

    n: int
    nt: int
    tile_rows: np.ndarray  # int32, (col,row) order
    tile_cols: np.ndarray  # int32
    _sym: _Sym | None = field(default=None, repr=False)
    _map: np.ndarray | None = field(default=None, repr=False)

    @property
    def tiles_per_side(self) -> int:
        return -(-self.n // self.nt)

    @property
    def n_tiles(self) -> int:
        return int(self.tile_rows.size)

    @property
    def slot_map(self) -> np.ndarray:
        if self._map is None:
            T = self.tiles_per_side
            sm = np.full((T, T), -1, dtype=np.int32)
            sm[self.tile_rows, self.tile_cols] = np.arange(self.n_tiles, dtype=np.int32)
            self._map = sm
        return self._map

    @property
    def keys(self) -> np.ndarray:
        """Sorted int64 keys col*T + row of the slots."""
        T = self.tiles_per_side
        return self.tile_cols.astype(np.int64) * T + self.tile_rows

    def slots_of(self, rows, cols) -> np.ndarray:
        """Vectorised slot lookup; -1 where not allocated (no dense map)."""
        T = self.tiles_per_side
        rr = np.asarray(rows, dtype=np.int64)
        cc = np.asarray(cols, dtype=np.int64)
        key = np.maximum(rr, cc) + T * np.minimum(rr, cc)
        keys = self.keys
        pos = np.searchsorted(keys, key)
        pos = np.minimum(pos, keys.size - 1)
        return np.where(keys[pos] == key, pos, -1).astype(np.int64)

    @property
    def occupancy(self) -> set:
        return {(int(r), int(c)) for r, c in zip(self.tile_rows, self.tile_cols)}

    def slot(self, r: int, c: int) -> int:
        s = int(self.slots_of([r], [c])[0]) if r >= c else -1
        if s < 0:
            raise KeyError(f"tile ({r}, {c}) is not allocated")
        return s

    def contains(self, r: int, c: int) -> bool:
        return r >= c and int(self.slots_of([r], [c])[0]) >= 0

    def occupancy_coordinates(self) -> str:
        return "\n".join(f"{r} {c}" for r, c in zip(self.tile_rows.tolist(), self.tile_cols.tolist()))


def grid_from_tiles(n: int, nt: int, rows, cols) -> TileGrid:
    """Occupied tiles (normalised to the lower triangle) + all diagonals
    (reference ctsf.py:57-75)."""
    T = -(-n // nt)
    r = np.asarray(rows, dtype=np.int64).ravel()
    c = np.asarray(cols, dtype=np.int64).ravel()
    key = np.concatenate([np.minimum(r, c) * T + np.maximum(r, c),
                          np.arange(T, dtype=np.int64) * (T + 1)])
    key = np.unique(key)
    return TileGrid(n=n, nt=nt, tile_rows=(key % T).astype(np.int32),
                    tile_cols=(key // T).astype(np.int32))


def build_tile_grid(m: SymmetricCsc, nt: int) -> TileGrid:
    """Tiles receiving a stored scalar + all diagonals (reference
    ctsf.py:78-84); computed in C++ (no nnz-length temporaries)."""
    if nt < 1:
        raise ValueError(f"tile size must be >= 1, got {nt}")
    sym = _sym_from_csc(m, nt)
    _, s_in, _, _ = sym.info()
    r = np.empty(s_in, dtype=np.int32)
    c = np.empty(s_in, dtype=np.int32)
    check("tc_symbolic_grid", lib.tc_symbolic_grid(sym.h, ptr(r, i32p), ptr(c, i32p)))
    return TileGrid(n=m.n, nt=nt, tile_rows=r, tile_cols=c, _sym=sym)


@dataclass(eq=False)
class TiledMatrix:
    """Dense tiles of the lower triangle (reference ctsf.py:87-115)."""

    grid: TileGrid
    storage: object  # numpy (S, nt, nt) or torch CUDA tensor

    @property
    def nt(self) -> int:
        return self.grid.nt

    def tile(self, r: int, c: int):
        return self.storage[self.grid.slot(r, c)].T

    def copy(self) -> "TiledMatrix":
        st = self.storage
        return TiledMatrix(grid=self.grid, storage=st.clone() if hasattr(st, "clone") else st.copy())

    def host_storage(self) -> np.ndarray:
        st = self.storage
        return st.detach().cpu().numpy() if hasattr(st, "detach") else st

    def get(self, i: int, j: int) -> float:
        if i < j:
            i, j = j, i
        nt = self.grid.nt
        return float(self.tile(i // nt, j // nt)[i % nt, j % nt])


def scatter_offsets(m: SymmetricCsc, grid: TileGrid) -> np.ndarray:
    """Flat storage offset of every stored scalar (slot*nt^2 + col*nt + row)."""
    nt = grid.nt
    cols = np.repeat(np.arange(m.n, dtype=np.int64), np.diff(m.col_ptr))
    rows = m.row_idx.astype(np.int64)
    slot = grid.slots_of(rows // nt, cols // nt)
    if slot.size and slot.min() < 0:
        raise ValueError("grid does not cover the matrix pattern")
    return slot * (nt * nt) + (cols % nt) * nt + rows % nt


def pack_into_grid(m: SymmetricCsc, grid: TileGrid) -> TiledMatrix:
    """Host scatter with unit padding on the last diagonal tile (reference
    ctsf.py:118-139).  The API path scatters on the device instead."""
    nt = grid.nt
    st = np.zeros((grid.n_tiles, nt, nt))
    st.reshape(-1)[scatter_offsets(m, grid)] = m.values
    lo = m.n % nt
    if lo:
        T = grid.tiles_per_side
        last = grid.slot(T - 1, T - 1)
        idx = np.arange(lo, nt)
        st[last, idx, idx] = 1.0
    return TiledMatrix(grid=grid, storage=st)


def pack_ctsf(m: SymmetricCsc, nt: int) -> TiledMatrix:
    return pack_into_grid(m, build_tile_grid(m, nt))


def expand_to_grid(t: TiledMatrix, grid: TileGrid) -> TiledMatrix:
    """Re-home tiles into a covering grid (reference ctsf.py:147-156)."""
    if grid.n_tiles == t.grid.n_tiles and np.array_equal(grid.keys, t.grid.keys):
        return t
    dst = grid.slots_of(t.grid.tile_rows, t.grid.tile_cols)
    if dst.size and dst.min() < 0:
        raise ValueError("target grid does not cover the source occupancy")
    src = t.host_storage()
    st = np.zeros((grid.n_tiles, grid.nt, grid.nt))
    st[dst] = src
    return TiledMatrix(grid=grid, storage=st)


def unpack_to_csc(t: TiledMatrix) -> SymmetricCsc:
    """Tiles -> CSC, dropping padding and exact zeros (reference ctsf.py:159-184)."""
    g, nt, n = t.grid, t.grid.nt, t.grid.n
    st = t.host_storage()
    j, i = np.meshgrid(np.arange(nt), np.arange(nt), indexing="ij")  # st[s, j, i]
    i = i.ravel()
    j = j.ravel()
    R, Cc, V = [], [], []
    for s in range(g.n_tiles):
        tr, tcol = int(g.tile_rows[s]), int(g.tile_cols[s])
        v = st[s].ravel()
        gi, gj = tr * nt + i, tcol * nt + j
        keep = (v != 0.0) & (gi < n) & (gj < n) & (gi >= gj)
        R.append(gi[keep])
        Cc.append(gj[keep])
        V.append(v[keep])
    return from_coordinates(n, np.concatenate(R), np.concatenate(Cc), np.concatenate(V),
                            sum_duplicates=False)
