"""Tile-level symbolic factorisation and planning (reference symbolic.py).

The elimination game, accumulation counts, the left-looking task stream,
tree-reduction plans and DAG statistics are computed by the C++ host library
(sparse etree form; no T x T boolean maps) and are bit-exact with the
reference.  Per-worker CPU task tables and DOT export are out of scope
(survey §2.1 row 5): the device launch plan replaces them.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field
from typing import NamedTuple

import numpy as np

from ._lib import check, i8p, i32p, i64p, lib, ptr
from .ctsf import TileGrid, _Sym, _sym_from_tiles

T_POTRF, T_SYRK, T_TRSM, T_GEMM, T_GEADD, T_ZERO = 1, 2, 3, 4, 5, 6
TYPE_NAMES = {1: "POTRF", 2: "SYRK", 3: "TRSM", 4: "GEMM", 5: "GEADD", 6: "ZERO"}

__all__ = ["T_POTRF", "T_SYRK", "T_TRSM", "T_GEMM", "T_GEADD", "T_ZERO", "TYPE_NAMES",
           "Task", "TaskList", "TileSymbolic", "tile_symbolic_factorize", "enumerate_tasks",
           "ReducedChain", "ReductionPlan", "plan_tree_reduction", "DagStats", "dag_stats"]


class Task(NamedTuple):
    m: int
    k: int
    n: int
    type: int


@dataclass(eq=False)
class TaskList:
    """Tasks as parallel arrays in execution order (reference symbolic.py:33-63)."""

    task_type: np.ndarray  # int8
    m: np.ndarray          # int32
    k: np.ndarray
    n: np.ndarray
    target: np.ndarray

    def __len__(self) -> int:
        return int(self.task_type.size)

    def __getitem__(self, i) -> Task:
        return Task(int(self.m[i]), int(self.k[i]), int(self.n[i]), int(self.task_type[i]))

    def take(self, positions) -> "TaskList":
        return TaskList(self.task_type[positions], self.m[positions], self.k[positions],
                        self.n[positions], self.target[positions])

    def counts_by_type(self) -> dict:
        counts = np.bincount(self.task_type.astype(np.int64), minlength=7)
        return {name: int(counts[code]) for code, name in TYPE_NAMES.items()
                if code <= 4 or counts[code]}

    def to_tuples(self) -> list:
        return [self[i] for i in range(len(self))]


@dataclass(eq=False)
class TileSymbolic:
    """Input grid, factor grid (input + fill) and per-slot accumulation
    counts (reference symbolic.py:66-95)."""

    grid: TileGrid
    factor_grid: TileGrid
    accum: np.ndarray
    _sym: _Sym = field(default=None, repr=False)

    @property
    def tiles_per_side(self) -> int:
        return self.grid.tiles_per_side

    @property
    def factor_occupancy(self) -> set:
        return self.factor_grid.occupancy

    def accum_count(self, m: int, k: int) -> int:
        return int(self.accum[self.factor_grid.slot(m, k)])

    def neighbors(self, k: int) -> np.ndarray:
        """Tiles m with factor tile (m, k) or (k, m) allocated, ascending."""
        fg = self.factor_grid
        in_col = fg.tile_rows[fg.tile_cols == k]
        in_row = fg.tile_cols[fg.tile_rows == k]
        return np.unique(np.concatenate([in_row, in_col]).astype(np.int64))


def tile_symbolic_factorize(g: TileGrid) -> TileSymbolic:
    """Tile elimination game (reference symbolic.py:98-123)."""
    sym = g._sym if g._sym is not None else _sym_from_tiles(g.n, g.nt, g.tile_rows, g.tile_cols)
    _, _, S, _ = sym.info()
    fr = np.empty(S, dtype=np.int32)
    fc = np.empty(S, dtype=np.int32)
    acc = np.empty(S, dtype=np.int64)
    check("tc_symbolic_factor", lib.tc_symbolic_factor(sym.h, ptr(fr, i32p), ptr(fc, i32p),
                                                       ptr(acc, i64p)))
    fg = TileGrid(n=g.n, nt=g.nt, tile_rows=fr, tile_cols=fc)
    return TileSymbolic(grid=g, factor_grid=fg, accum=acc, _sym=sym)


def _sym_of(s: TileSymbolic) -> _Sym:
    if s._sym is None:
        s._sym = _sym_from_tiles(s.grid.n, s.grid.nt, s.grid.tile_rows, s.grid.tile_cols)
    return s._sym


def enumerate_tasks(s: TileSymbolic) -> TaskList:
    """Left-looking stream: per k, SYRKs by ascending n, POTRF(k), then per
    m > k its GEMMs by ascending n and its TRSM (reference symbolic.py:126-164)."""
    sym = _sym_of(s)
    _, _, _, P = sym.info()
    ty = np.empty(P, dtype=np.int8)
    m, k, n, tg = (np.empty(P, dtype=np.int32) for _ in range(4))
    check("tc_symbolic_tasks", lib.tc_symbolic_tasks(sym.h, ptr(ty, i8p), ptr(m, i32p), ptr(k, i32p),
                                                     ptr(n, i32p), ptr(tg, i32p)))
    return TaskList(task_type=ty, m=m, k=k, n=n, target=tg)


@dataclass(frozen=True)
class ReducedChain:
    slot: int
    ranges: tuple
    combine: tuple


@dataclass(eq=False)
class ReductionPlan:
    workers: int
    chains: dict = field(default_factory=dict)

    def __bool__(self) -> bool:
        return bool(self.chains)

    def chain_for_tile(self, s: TileSymbolic, m: int, k: int):
        return self.chains.get(s.factor_grid.slot(m, k))


def _combine_steps(r: int) -> tuple:
    """Pairwise GEADD tree (a, a + stride), stride doubling
    (reference symbolic.py:241-250)."""
    out = []
    stride = 1
    while stride < r:
        out += [(a, a + stride) for a in range(0, r - stride, 2 * stride)]
        stride <<= 1
    return tuple(out)


def plan_tree_reduction(s: TileSymbolic, workers: int) -> ReductionPlan:
    """Split chains with accum >= 2*workers into near-equal contiguous ranges
    (reference symbolic.py:253-269)."""
    if workers < 2:
        raise ValueError("tree reduction needs at least 2 workers")
    sym = _sym_of(s)
    cnt = np.zeros(1, dtype=np.int64)
    check("tc_symbolic_tree_plan", lib.tc_symbolic_tree_plan(sym.h, workers, ptr(cnt, i64p), None, None))
    c = int(cnt[0])
    slots = np.empty(c, dtype=np.int64)
    ranges = np.empty((c, workers, 2), dtype=np.int64)
    check("tc_symbolic_tree_plan", lib.tc_symbolic_tree_plan(sym.h, workers, ptr(cnt, i64p),
                                                             ptr(slots, i64p), ptr(ranges, i64p)))
    comb = _combine_steps(workers)
    plan = ReductionPlan(workers=workers)
    for i, sl in enumerate(slots.tolist()):
        plan.chains[sl] = ReducedChain(slot=sl, ranges=tuple(map(tuple, ranges[i].tolist())),
                                       combine=comb)
    return plan


@dataclass(frozen=True)
class DagStats:
    counts: dict
    total_tasks: int
    critical_path: int
    max_width: int

    def to_json(self) -> str:
        return json.dumps({"counts": self.counts, "total_tasks": self.total_tasks,
                           "critical_path": self.critical_path, "max_width": self.max_width})


def dag_stats(s: TileSymbolic) -> DagStats:
    """Task counts, unit-cost critical path and widest level (reference
    symbolic.py:287-331)."""
    sym = _sym_of(s)
    cp = np.zeros(1, dtype=np.int64)
    w = np.zeros(1, dtype=np.int64)
    check("tc_symbolic_dag_stats", lib.tc_symbolic_dag_stats(sym.h, ptr(cp, i64p), ptr(w, i64p)))
    tasks = enumerate_tasks(s)
    return DagStats(counts=tasks.counts_by_type(), total_tasks=len(tasks),
                    critical_path=int(cp[0]), max_width=int(w[0]))


def compile_ops(s: TileSymbolic, workers: int = 0):
    """Op arrays (op_type int8, dst, src1, src2 int64) and scratch count for
    ``run_ops``: the reconstruction of the reference's missing scheduler op
    compiler, tree-reduced for chains >= 2*workers when
    workers >= 2."""
    sym = _sym_of(s)
    P = np.zeros(1, dtype=np.int64)
    R = np.zeros(1, dtype=np.int64)
    check("tc_symbolic_compile_ops", lib.tc_symbolic_compile_ops(sym.h, workers, ptr(P, i64p), ptr(R, i64p),
                                                                 None, None, None, None))
    n = int(P[0])
    op = np.empty(n, dtype=np.int8)
    dst, s1, s2 = (np.empty(n, dtype=np.int64) for _ in range(3))
    check("tc_symbolic_compile_ops", lib.tc_symbolic_compile_ops(
        sym.h, workers, ptr(P, i64p), ptr(R, i64p), ptr(op, i8p), ptr(dst, i64p), ptr(s1, i64p),
        ptr(s2, i64p)))
    return op, dst, s1, s2, int(R[0])
