"""Device launch plan — the B200 replacement of the reference's (missing)
static scheduler (paper Alg. 1-3).

The plan is built once per factor tile pattern in C++ (``tc_plan_create``):

* column step k = bulk update B(k) (all left-looking contributions except the
  last one, lookahead), last update L(k), POTRF(k), TRSM(k);
* chains with accum >= 2W (the arrow x arrow tiles) are split-K over W
  partial tiles filled as the band factorisation proceeds and combined by the
  deterministic pairwise tree of symbolic._combine_steps (Alg. 3);
* the launches form a dependency DAG, executed either by the persistent
  dataflow kernel (default: one launch, tasks handed out by a device ticket
  counter in a topological priority order, per-launch dependency counters —
  the device form of the paper's progress table) or as one CUDA graph per
  lane with critical-path nodes at high stream priority.

``compile_ops`` (the reference-compatible op stream for ``run_ops``) lives in
symbolic.py.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import PlanOpts, check, f64p, i32p, i64p, lib, ptr
from .ctsf import TileGrid

__all__ = ["PlanOptions", "DevicePlan"]


@dataclass(frozen=True)
class PlanOptions:
    tree_workers: int = 8        # W partial accumulators per long chain
    tree_threshold: int = 0      # 0 = 2*W (reference rule), < 0 = no tree reduction
    chunk: int = 0               # columns per split-K launch (0 = 8)
    lookahead: int = -1          # columns of lookahead for the bulk update (-1 = auto, 0 = off)
    executor: str = "persistent"  # persistent | graph | direct
    occupancy: int = 0            # persistent CTAs per SM: 0 auto (2 when it fits), 1, 2
    fuse_trsm: bool = True        # persistent: TRSM(k) streams POTRF(k)'s panels
    concurrent: int = 1           # persistent: factorisations sharing the GPU (grid share)

    def to_c(self) -> PlanOpts:
        o = PlanOpts()
        o.tree_workers = self.tree_workers
        o.tree_threshold = self.tree_threshold
        o.chunk = self.chunk
        o.lookahead = int(self.lookahead)
        o.use_graph = {"direct": 0, "graph": 1, "persistent": 2}[self.executor]
        o.reserved[0] = 0 if self.fuse_trsm else 1
        o.reserved[1] = int(self.occupancy)
        o.reserved[2] = int(self.concurrent)
        return o


class DevicePlan:
    """Owner of a ``tc_plan_t`` for one (n, nt, factor pattern)."""

    def __init__(self, factor_grid: TileGrid, options: PlanOptions | None = None):
        _lib.require_device()
        self.grid = factor_grid
        self.n, self.nt = factor_grid.n, factor_grid.nt
        self.T = factor_grid.tiles_per_side
        self.S = factor_grid.n_tiles
        self.options = options or PlanOptions()
        r = _lib.i32arr(factor_grid.tile_rows)
        c = _lib.i32arr(factor_grid.tile_cols)
        h = C.c_void_p()
        opts = self.options.to_c()
        check("tc_plan_create", lib.tc_plan_create(self.n, self.nt, self.S, ptr(r, i32p), ptr(c, i32p),
                                                   C.byref(opts), C.byref(h)))
        self.h = h

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            lib.tc_plan_destroy(h)
            self.h = C.c_void_p(0)

    def info(self) -> dict:
        a, b, c, d = (np.zeros(1, dtype=np.int64) for _ in range(4))
        f = np.zeros(1, dtype=np.float64)
        check("tc_plan_info", lib.tc_plan_info(self.h, ptr(a, i64p), ptr(b, i64p), ptr(c, i64p),
                                               ptr(d, i64p), ptr(f, f64p)))
        return {"launches": int(a[0]), "items": int(b[0]), "pairs": int(c[0]),
                "scratch_tiles": int(d[0]), "tile_flops": float(f[0])}

    # ---- device buffers -------------------------------------------------
    def new_storage(self):
        import torch
        return torch.empty((self.S, self.nt, self.nt), dtype=torch.float64, device="cuda")

    def offsets_for(self, m) -> np.ndarray:
        """Flat storage offsets of m's stored scalars (host).  Not cached here:
        the caller (api._Pattern) owns the pattern and caches its offsets."""
        off = np.empty(m.nnz, dtype=np.int64)
        cp, ri = _lib.i64arr(m.col_ptr), _lib.i32arr(m.row_idx)
        check("tc_plan_pack_offsets", lib.tc_plan_pack_offsets(self.h, m.n, ptr(cp, i64p), ptr(ri, i32p),
                                                               ptr(off, i64p)))
        return off

    def pack_lincomb(self, basis_dev, coef, offsets_dev, storage, stream: int) -> None:
        """storage <- scatter of sum_i coef[i] * basis_dev[i] (device value
        assembly of one member of a matrix family on this pattern)."""
        c = np.ascontiguousarray(np.asarray(coef, dtype=np.float64))
        check("tc_plan_pack_lincomb", lib.tc_plan_pack_lincomb(
            self.h, basis_dev.data_ptr(), int(basis_dev.shape[0]), ptr(c, f64p), offsets_dev.data_ptr(),
            int(basis_dev.shape[1]), storage.data_ptr(), stream))

    def pack(self, values_dev, offsets_dev, storage, stream: int) -> None:
        """Zero storage, scatter values (device), unit-pad the last diagonal."""
        check("tc_plan_pack", lib.tc_plan_pack(self.h, values_dev.data_ptr(), offsets_dev.data_ptr(),
                                               int(values_dev.numel()), storage.data_ptr(), stream))

    # ---- numeric phase --------------------------------------------------
    def factorize_async(self, storage, lane: int, stream: int) -> None:
        check("tc_plan_factorize_async", lib.tc_plan_factorize_async(self.h, lane, storage.data_ptr(), stream))

    def copy_result(self, lane: int, stream: int, fail_dev, logdet_dev) -> None:
        """Enqueue device copies of the lane's failure word / log-determinant
        (int64 / float64 device tensors of one element, e.g. views into a batch array)."""
        check("tc_plan_copy_result", lib.tc_plan_copy_result(self.h, lane, stream, fail_dev.data_ptr(),
                                                             logdet_dev.data_ptr()))

    def collect(self, lane: int, stream: int):
        f = np.zeros(1, dtype=np.int64)
        ld = np.zeros(1, dtype=np.float64)
        check("tc_plan_collect", lib.tc_plan_collect(self.h, lane, stream, ptr(f, i64p), ptr(ld, f64p)))
        return int(f[0]), float(ld[0])

    def factorize(self, storage, lane: int = 0, stream: int | None = None):
        """In-place factorisation; returns (fail_index or -1, logdet)."""
        s = _current_stream() if stream is None else stream
        self.factorize_async(storage, lane, s)
        return self.collect(lane, s)

    def logdet(self, storage, stream: int | None = None) -> float:
        out = np.zeros(1, dtype=np.float64)
        s = _current_stream() if stream is None else stream
        check("tc_plan_logdet", lib.tc_plan_logdet(self.h, storage.data_ptr(), s, ptr(out, f64p)))
        return float(out[0])

    def solve(self, storage, rhs_dev, stream: int | None = None) -> None:
        """In place: rhs_dev (nrhs, T*nt) <- L^-T L^-1 rhs_dev (permuted domain)."""
        s = _current_stream() if stream is None else stream
        check("tc_plan_solve", lib.tc_plan_solve(self.h, storage.data_ptr(), rhs_dev.data_ptr(),
                                                 int(rhs_dev.shape[0]), s))


def _current_stream() -> int:
    import torch
    return torch.cuda.current_stream().cuda_stream
