"""CPU oracle for the sTiles / tilechol arrowhead tile-Cholesky path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2501_02483_b200`` may import
this package; only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` use it, and only
as the checker (or as the timed *reference* CPU arm), never as the product.

It is a from-scratch CPU restatement of the reference algorithm (each
function cites the reference file:line it follows).  It is *pinned* against
golden vectors produced by the live reference (``tests/golden/make_golden.py``
imports ``/root/reference/pkg/src/tilechol`` in the build container and
commits the fixtures); ``tests/test_oracle_golden.py`` checks every fixture.
"""

from .core import *  # noqa: F401,F403
