"""The C-ABI library loads and exports every symbol include/*.h declares."""
import ctypes
import glob
import os
import re

from conftest import ROOT


def test_library_exports_every_declared_symbol():
    from paper_2501_02483_b200 import _lib
    decl = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        txt = open(h).read()
        txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
        decl |= set(re.findall(r"\b(tc_[a-z0-9_]+)\s*\(", txt))
    assert len(decl) >= 35
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in sorted(decl) if not hasattr(lib, s)]
    assert not missing, missing
    assert set(_lib.SIGNATURES) == decl


def test_no_gpu_means_loud_failure_not_fallback():
    from paper_2501_02483_b200 import _lib
    if _lib.device_count() > 0:
        return
    import numpy as np
    import pytest
    from paper_2501_02483_b200.backend import impl
    with pytest.raises(RuntimeError, match="no CUDA device"):
        impl.potrf_tile(np.eye(4, order="F"))
