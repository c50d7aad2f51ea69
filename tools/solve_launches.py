"""One C2 factorisation + one device solve (1 RHS), for an ncu launch list of
the solve phases (batched L_kk^-T TRSM, sweep):
    ncu --metrics gpu__time_duration.sum --csv python tools/solve_launches.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2501_02483_b200 import api  # noqa: E402

m = bench.build_matrix(sys.argv[1] if len(sys.argv) > 1 else "c2")
ctx = api.factorize(m, api.FactorOptions(tile_size=128))
plan = ctx.plan
r = torch.ones((1, plan.T * plan.nt), dtype=torch.float64, device="cuda")
plan.solve(ctx.factor.storage, r)
torch.cuda.synchronize()
print("ok", float(r.sum()))
