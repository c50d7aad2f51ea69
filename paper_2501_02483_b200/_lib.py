"""ctypes binding of ``libtilechol_b200.so`` (the C ABI in include/tilechol_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2501_02483_b200/csrc``).  There is no fallback: importing this
module without the library raises ImportError, and device entry points raise
RuntimeError when no CUDA device is visible.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TILECHOL_B200_LIB", os.path.join(_HERE, "libtilechol_b200.so"))

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"libtilechol_b200.so not found at {LIB_PATH}; build it with "
        "`python -c 'import __graft_entry__ as g; g.build()'` or "
        "`make -C paper_2501_02483_b200/csrc`")

lib = C.CDLL(LIB_PATH)

i8p = C.POINTER(C.c_int8)
u8p = C.POINTER(C.c_uint8)
i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)
vp = C.c_void_p
i32, i64, f64 = C.c_int32, C.c_int64, C.c_double

TC_OK = 0
OP_POTRF, OP_SYRK, OP_TRSM, OP_GEMM, OP_GEADD, OP_ZERO = 1, 2, 3, 4, 5, 6


class PlanOpts(C.Structure):
    _fields_ = [("tree_workers", i32), ("tree_threshold", i32), ("chunk", i32),
                ("lookahead", i32), ("use_graph", i32), ("reserved", i32 * 3)]


# name -> (restype, argtypes); every symbol declared in include/tilechol_b200.h
SIGNATURES = {
    "tc_last_error": (C.c_char_p, []),
    "tc_abi_version": (i32, []),
    "tc_device_count": (i32, []),
    "tc_etree_fill_count": (C.c_int, [i64, i64p, i64p, i64p]),
    "tc_symbolic_fill_count": (C.c_int, [i64, i64p, i32p, i64p, i64p]),
    "tc_zero_fill": (C.c_int, [i64, i64p, i32p, i32p, i64p]),
    "tc_structure_stats": (C.c_int, [i64, i64p, i32p, f64, i64p, i64p]),
    "tc_factor_column_counts": (C.c_int, [i64, i64p, i32p, i64p, i64p]),
    "tc_arrowhead_pattern": (C.c_int, [i64, i64, i64, i32, i64p, i32p]),
    "tc_arrowhead_diag": (C.c_int, [i64, i64p, i32p, f64p]),
    "tc_band_arrow_pattern": (C.c_int, [i64, i64, i64p, i64p, i32p]),
    "tc_rcm": (C.c_int, [i64, i64p, i32p, i64, i64p]),
    "tc_adaptable_nd": (C.c_int, [i64, i64, i64, i32, i64p]),
    "tc_symbolic_from_csc": (C.c_int, [i64, i32, i64p, i32p, C.POINTER(vp)]),
    "tc_symbolic_from_tiles": (C.c_int, [i64, i32, i64, i64p, i64p, C.POINTER(vp)]),
    "tc_symbolic_info": (C.c_int, [vp, i64p, i64p, i64p, i64p]),
    "tc_symbolic_grid": (C.c_int, [vp, i32p, i32p]),
    "tc_symbolic_factor": (C.c_int, [vp, i32p, i32p, i64p]),
    "tc_symbolic_tasks": (C.c_int, [vp, i8p, i32p, i32p, i32p, i32p]),
    "tc_symbolic_tree_plan": (C.c_int, [vp, i32, i64p, i64p, i64p]),
    "tc_symbolic_compile_ops": (C.c_int, [vp, i32, i64p, i64p, i8p, i64p, i64p, i64p]),
    "tc_symbolic_dag_stats": (C.c_int, [vp, i64p, i64p]),
    "tc_symbolic_destroy": (None, [vp]),
    "tc_potrf_tile": (C.c_int, [vp, i32, vp, i32p]),
    "tc_trsm_tile": (C.c_int, [vp, vp, i32, vp, i32p]),
    "tc_syrk_tile": (C.c_int, [vp, vp, i32, vp]),
    "tc_gemm_tile": (C.c_int, [vp, vp, vp, i32, vp]),
    "tc_geadd_tile": (C.c_int, [vp, vp, i32, vp]),
    "tc_run_ops": (C.c_int, [vp, i64, vp, i64, i32, i8p, i64p, i64p, i64p, i64, i64, i64, vp,
                             i64p, i32p]),
    "tc_replay_residual": (C.c_int, [vp, vp, i64, i32, i8p, i64p, i64p, i64p, i64, u8p, vp,
                                     f64p]),
    "tc_plan_create": (C.c_int, [i64, i32, i64, i32p, i32p, C.POINTER(PlanOpts), C.POINTER(vp)]),
    "tc_plan_info": (C.c_int, [vp, i64p, i64p, i64p, i64p, f64p]),
    "tc_plan_factorize": (C.c_int, [vp, vp, vp, i64p]),
    "tc_plan_factorize_async": (C.c_int, [vp, i32, vp, vp]),
    "tc_plan_collect": (C.c_int, [vp, i32, vp, i64p, f64p]),
    "tc_plan_copy_result": (C.c_int, [vp, i32, vp, vp, vp]),
    "tc_plan_debug_ticket": (C.c_int, [vp, i32, i32p, i32p]),
    "tc_host_register": (C.c_int, [vp, C.c_size_t]),
    "tc_host_unregister": (C.c_int, [vp]),
    "tc_memcpy_h2d_async": (C.c_int, [vp, vp, C.c_size_t, vp]),
    "tc_plan_logdet": (C.c_int, [vp, vp, vp, f64p]),
    "tc_plan_solve": (C.c_int, [vp, vp, vp, i32, vp]),
    "tc_plan_pack_offsets": (C.c_int, [vp, i64, i64p, i32p, i64p]),
    "tc_plan_pack": (C.c_int, [vp, vp, vp, i64, vp, vp]),
    "tc_plan_pack_lincomb": (C.c_int, [vp, vp, i32, f64p, vp, i64, vp, vp]),
    "tc_plan_destroy": (None, [vp]),
    "tc_plan_profile": (C.c_int, [vp, vp, vp, i32, f64p, i64p, f64p]),
    "tc_plan_trace": (C.c_int, [vp, vp, vp, i64, i64p, i32p, i64, i32p, i64p, i64p]),
    "tc_bench_dmma_peak": (C.c_int, [i64, i32, i32, f64p]),
}

for _name, (_res, _args) in SIGNATURES.items():
    if "TILECHOL_B200_LIB" in os.environ and not hasattr(lib, _name):
        continue  # A/B runs against an older build (tools/ab.sh)
    _f = getattr(lib, _name)  # AttributeError here = stale/foreign library
    _f.restype = _res
    _f.argtypes = _args


class TcError(RuntimeError):
    """A C-ABI call returned a non-zero status."""

    def __init__(self, fn, code):
        self.code = code
        msg = lib.tc_last_error().decode(errors="replace")
        super().__init__(f"{fn} failed (status {code}): {msg}")


def check(fn, code):
    if code != TC_OK:
        if code == -1:
            raise ValueError(f"{fn}: {lib.tc_last_error().decode(errors='replace')}")
        raise TcError(fn, code)


def ptr(a: np.ndarray, ctype):
    """ctypes pointer to a contiguous numpy array (None for None)."""
    if a is None:
        return None
    return a.ctypes.data_as(ctype)


def i64arr(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.int64))


def i32arr(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.int32))


def device_count() -> int:
    return int(lib.tc_device_count())


def require_device():
    if device_count() < 1:
        raise RuntimeError("tilechol_b200: no CUDA device visible; the B200 path has no CPU fallback")
