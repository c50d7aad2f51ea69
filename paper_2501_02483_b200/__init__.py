"""paper_2501_02483_b200 — B200-native sTiles arrowhead tile Cholesky.

A drop-in for the reference ``tilechol`` hot path: the ``backend.impl`` plugin
seam (8 functions), the host preprocessing it consumes (orderings, tile
symbolic, task stream; bit-exact), and the SPEC api (factorize / solve /
logdet / factorize_many).  Numerics are hand-written sm_100a FP64 kernels
(DMMA) driven by a CUDA-graph launch plan; see DESIGN.md.
"""

from . import backend, ctsf, errors, matcore, ordering, scheduler, symbolic  # noqa: F401
from .api import (FactorContext, FactorOptions, clear_plan_cache, factorize,  # noqa: F401
                  factorize_many, factorize_many_sharded, logdet, solve)
from .errors import (FactorizeManyError, MatrixFormatError, NotPositiveDefiniteError,  # noqa: F401
                     TileCholError)
from .matcore import ArrowheadSpec, SymmetricCsc, generate_arrowhead  # noqa: F401

__version__ = "0.1.0"
