"""Backend seam (reference backend.py:1-26).

``impl`` exposes potrf_tile, trsm_tile, syrk_tile, gemm_tile, geadd_tile,
run_ops, replay_residual and etree_fill_count.  Unlike the reference there is
one implementation only — the sm_100a kernels in libtilechol_b200.so — and no
silent fallback: a missing library fails at import.
"""

from . import _backend_cuda as impl  # noqa: F401

BACKEND = "cuda-sm100a"
