"""Repeat one factorisation; report the first differing tile vs the first run."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_2501_02483_b200 import api
name, nt, reps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
occ = int(sys.argv[4]) if len(sys.argv) > 4 else 0
m = bench.build_matrix(name)
opts = api.FactorOptions(tile_size=nt, occupancy=occ, ordering="identity")
pat = api._pattern_for(m, opts)
plan = pat.plan
fg = pat.symbolic.factor_grid
rows, cols = np.asarray(fg.tile_rows), np.asarray(fg.tile_cols)
vals = torch.from_numpy(np.ascontiguousarray(pat.permuted_values(m))).cuda()
st = plan.new_storage()
sh = torch.cuda.current_stream().cuda_stream
ref = None
for r in range(reps):
    plan.pack(vals, pat.offsets(), st, sh)
    plan.factorize_async(st, 0, sh)
    f, ld = plan.collect(0, sh)
    if ref is None:
        ref = st.clone()
        ld0 = ld
        continue
    d = (st != ref).flatten(1).any(dim=1)
    bad = torch.nonzero(d).flatten().cpu().numpy()
    if bad.size == 0:
        print(f"rep {r}: identical", flush=True)
        continue
    # first differing tile in factorisation order (column, then row)
    order = np.lexsort((rows[bad], cols[bad]))
    b0 = bad[order[0]]
    diff = (st[b0] - ref[b0]).abs()
    idx = int(torch.argmax(diff).item())
    print(f"rep {r}: {bad.size} tiles differ, ld diff {ld - ld0:.3e}; first tile slot {b0} "
          f"({rows[b0]},{cols[b0]}) max {diff.max().item():.3e} at storage[{idx // nt},{idx % nt}] "
          f"(col {idx // nt}, row {idx % nt}); arrow rows >= {(m.n - 1) // nt}", flush=True)
