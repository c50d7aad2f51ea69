"""Diagnostic: factorise one workload at occupancy 1 and at occupancy 2 (same
plan options otherwise) and report the first differing factor slots (column
order), per-column max relative difference and the logdets.

    TILECHOL_EXPERIMENTAL=1 python tools/occ_diff.py --workload c4 [--tree off] [--lookahead 1]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["TILECHOL_EXPERIMENTAL"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2501_02483_b200 import api  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c4")
ap.add_argument("--tile", type=int, default=120)
ap.add_argument("--tree", default="auto")
ap.add_argument("--lookahead", type=int, default=2)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--chain", type=int, default=1)
a = ap.parse_args()
m = bench.build_matrix(a.workload)
res = {}
for occ in (1, 2):
    opts = api.FactorOptions(tile_size=a.tile, ordering="identity", occupancy=occ, tree_reduction=a.tree,
                             lookahead=a.lookahead)
    pat = api._pattern_for(m, opts)
    plan = pat.plan
    vals = torch.from_numpy(np.ascontiguousarray(pat.permuted_values(m))).cuda()
    st = plan.new_storage()
    sh = torch.cuda.current_stream().cuda_stream
    lds = []
    for r in range(a.reps):
        plan.pack(vals, pat.offsets(), st, sh)
        plan.factorize_async(st, 0, sh)
        f, ld = plan.collect(0, sh)
        lds.append(ld)
    res[occ] = (st, lds, pat)
    print(f"occ {occ}: logdets {lds} fail {f}", flush=True)
    del vals
s1, s2 = res[1][0], res[2][0]
fg = res[1][2].symbolic.factor_grid
d = (s1 - s2).abs().amax(dim=(1, 2))
nz = torch.nonzero(d > 0).flatten().cpu().numpy()
print(f"slots differing: {nz.size} of {s1.shape[0]}")
if nz.size:
    rows, cols = fg.tile_rows[nz], fg.tile_cols[nz]
    for i in range(min(20, nz.size)):
        s = nz[i]
        rel = float(d[s] / s1[s].abs().max())
        print(f"  slot {s}: tile ({rows[i]}, {cols[i]}) max|diff| {float(d[s]):.3e} rel {rel:.3e}")
    print("first differing column", int(cols.min()), "rows there:", sorted(set(rows[cols == cols.min()].tolist())))
