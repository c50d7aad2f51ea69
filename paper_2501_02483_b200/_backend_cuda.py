"""B200 implementation of the reference plugin seam ``backend.impl``
(reference backend.py:1-26; contracts _backend_numba.py:16-215).

Exactly the eight reference functions, same argument meaning, in-place
mutation and return codes.  Arrays may be host numpy arrays (copied to the
GPU and back, like a drop-in for the numba backend) or CUDA torch tensors
(operated on in place).  Tiles are ``(nt, nt)`` column-major views, i.e.
``storage[s].T`` of a C-order ``(S, nt, nt)`` storage.  Every numeric call
runs an sm_100a kernel from ``libtilechol_b200.so``; there is no CPU path.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from ._lib import check, f64p, i8p, i32p, i64p, lib, ptr, u8p

POTRF, SYRK, TRSM, GEMM, GEADD, ZERO = 1, 2, 3, 4, 5, 6

__all__ = ["potrf_tile", "trsm_tile", "syrk_tile", "gemm_tile", "geadd_tile", "run_ops",
           "replay_residual", "etree_fill_count"]


def _torch():
    import torch
    _lib.require_device()
    return torch


def _stream():
    torch = _torch()
    return torch.cuda.current_stream().cuda_stream


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


class _Tile:
    """Device view of one column-major nt x nt tile."""

    def __init__(self, a, write_back: bool):
        torch = _torch()
        self.src = a
        self.wb = write_back
        if _is_torch(a):
            if not a.is_cuda or a.dtype != torch.float64:
                raise TypeError("tile tensors must be float64 CUDA tensors")
            nt = a.shape[0]
            if a.shape != (nt, nt) or a.stride() != (1, nt):
                raise ValueError("tile tensor must be a column-major (nt, nt) view, e.g. storage[s].T")
            self.dev = a
            self.host = False
        else:
            arr = np.asarray(a)
            if arr.dtype != np.float64 or arr.ndim != 2 or arr.shape[0] != arr.shape[1]:
                raise ValueError("tiles must be square float64 arrays")
            flat = np.asfortranarray(arr).reshape(-1, order="F")
            self.dev = torch.from_numpy(np.ascontiguousarray(flat)).cuda()
            self.host = True
        self.nt = int(a.shape[0])

    @property
    def ptr(self) -> int:
        return self.dev.data_ptr()

    def done(self):
        if self.host and self.wb:
            self.src[...] = self.dev.cpu().numpy().reshape(self.nt, self.nt, order="F")


def potrf_tile(a) -> int:
    """In-place lower Cholesky; -1 or first pivot index with a[j,j] <= 0."""
    t = _Tile(a, True)
    info = np.zeros(1, dtype=np.int32)
    check("tc_potrf_tile", lib.tc_potrf_tile(t.ptr, t.nt, _stream(), ptr(info, i32p)))
    if info[0] < 0:
        t.done()
    return int(info[0])


def trsm_tile(l, x) -> int:
    """Solve X L^T = B in place (B in x); -1 or first zero diagonal of l."""
    tl, tx = _Tile(l, False), _Tile(x, True)
    if tl.nt != tx.nt:
        raise ValueError("tile size mismatch")
    info = np.zeros(1, dtype=np.int32)
    check("tc_trsm_tile", lib.tc_trsm_tile(tl.ptr, tx.ptr, tl.nt, _stream(), ptr(info, i32p)))
    if info[0] < 0:
        tx.done()
    return int(info[0])


def syrk_tile(a, c) -> None:
    """c -= a a^T over the full tile."""
    ta, tc_ = _Tile(a, False), _Tile(c, True)
    check("tc_syrk_tile", lib.tc_syrk_tile(ta.ptr, tc_.ptr, ta.nt, _stream()))
    tc_.done()


def gemm_tile(a, b, c) -> None:
    """c -= b a^T."""
    ta, tb, tc_ = _Tile(a, False), _Tile(b, False), _Tile(c, True)
    check("tc_gemm_tile", lib.tc_gemm_tile(ta.ptr, tb.ptr, tc_.ptr, ta.nt, _stream()))
    tc_.done()


def geadd_tile(t, c) -> None:
    """c += t."""
    tt, tc_ = _Tile(t, False), _Tile(c, True)
    check("tc_geadd_tile", lib.tc_geadd_tile(tt.ptr, tc_.ptr, tt.nt, _stream()))
    tc_.done()


def _storage_dev(st, name):
    torch = _torch()
    if _is_torch(st):
        if not st.is_cuda or st.dtype != torch.float64 or not st.is_contiguous() or st.dim() != 3:
            raise ValueError(f"{name} must be a contiguous float64 CUDA tensor (S, nt, nt)")
        return st, False
    arr = np.asarray(st)
    if arr.dtype != np.float64 or arr.ndim != 3 or not arr.flags.c_contiguous:
        raise ValueError(f"{name} must be a C-contiguous float64 array (S, nt, nt)")
    return torch.from_numpy(arr).cuda(), True


def _ops(op_type, dst, src1, src2):
    op = np.ascontiguousarray(np.asarray(op_type, dtype=np.int8))
    d = _lib.i64arr(dst)
    a = _lib.i64arr(src1)
    b = _lib.i64arr(src2)
    if not (op.size == d.size == a.size == b.size):
        raise ValueError("op arrays must have equal length")
    return op, d, a, b


def run_ops(storage, scratch, op_type, dst, src1, src2, start, stop):
    """Execute ops [start, stop) in order; (stop, -1) or (p, info) at the first
    non-positive POTRF pivot / zero TRSM diagonal (later ops are skipped)."""
    op, d, a, b = _ops(op_type, dst, src1, src2)
    st, st_host = _storage_dev(storage, "storage")
    S, nt = int(st.shape[0]), int(st.shape[1])
    sc_host = False
    sc_ptr, R = None, 0
    if scratch is not None and int(scratch.shape[0]) > 0:
        sc, sc_host = _storage_dev(scratch, "scratch")
        sc_ptr, R = sc.data_ptr(), int(sc.shape[0])
    p = np.zeros(1, dtype=np.int64)
    info = np.zeros(1, dtype=np.int32)
    check("tc_run_ops", lib.tc_run_ops(st.data_ptr(), S, sc_ptr, R, nt, ptr(op, i8p), ptr(d, i64p),
                                       ptr(a, i64p), ptr(b, i64p), op.size, int(start), int(stop),
                                       _stream(), ptr(p, i64p), ptr(info, i32p)))
    if st_host:
        storage[...] = st.cpu().numpy()
    if sc_host:
        scratch[...] = sc.cpu().numpy()
    return int(p[0]), int(info[0])


def replay_residual(storage, template, op_type, dst, src1, src2, diag_slot) -> float:
    """Sum of squared errors of L L^T against the packed original over the
    sequential stream's target groups (symmetric weights)."""
    op, d, a, b = _ops(op_type, dst, src1, src2)
    st, _ = _storage_dev(storage, "storage")
    tp, _ = _storage_dev(template, "template")
    if tuple(st.shape) != tuple(tp.shape):
        raise ValueError("storage/template shape mismatch")
    dg = np.ascontiguousarray(np.asarray(diag_slot).astype(np.uint8))
    if dg.size != st.shape[0]:
        raise ValueError("diag_slot length must equal the slot count")
    out = np.zeros(1, dtype=np.float64)
    check("tc_replay_residual", lib.tc_replay_residual(
        st.data_ptr(), tp.data_ptr(), int(st.shape[0]), int(st.shape[1]), ptr(op, i8p), ptr(d, i64p),
        ptr(a, i64p), ptr(b, i64p), op.size, ptr(dg, u8p), _stream(), ptr(out, f64p)))
    return float(out[0])


def etree_fill_count(n, row_ptr, row_cols) -> int:
    """Strict-lower nnz(L) from a strict-lower CSR (host C++, no GPU)."""
    rp = _lib.i64arr(row_ptr)
    rc = _lib.i64arr(row_cols)
    out = np.zeros(1, dtype=np.int64)
    check("tc_etree_fill_count", lib.tc_etree_fill_count(int(n), ptr(rp, i64p), ptr(rc, i64p),
                                                         ptr(out, i64p)))
    return int(out[0])
