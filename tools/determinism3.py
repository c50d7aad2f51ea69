"""Back-to-back factorisations of one matrix (no sync between them) vs a synced reference."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_2501_02483_b200 import api
name, nt = sys.argv[1], int(sys.argv[2])
m = bench.build_matrix(name)
opts = api.FactorOptions(tile_size=nt, ordering="identity")
pat = api._pattern_for(m, opts)
plan = pat.plan
fg = pat.symbolic.factor_grid
rows, cols = np.asarray(fg.tile_rows), np.asarray(fg.tile_cols)
vals = torch.from_numpy(np.ascontiguousarray(pat.permuted_values(m))).cuda()
st = plan.new_storage()
sh = torch.cuda.current_stream().cuda_stream
def step():
    plan.pack(vals, pat.offsets(), st, sh)
    plan.factorize_async(st, 0, sh)
step(); plan.collect(0, sh)
ref = st.clone()
for trial in range(4):
    for _ in range(3):
        step()
    f, ld = plan.collect(0, sh)
    d = (st != ref).flatten(1).any(dim=1)
    bad = torch.nonzero(d).flatten().cpu().numpy()
    if bad.size == 0:
        print(f"trial {trial}: identical", flush=True)
        continue
    order = np.lexsort((rows[bad], cols[bad]))
    b0 = bad[order[0]]
    diff = (st[b0] - ref[b0]).abs()
    print(f"trial {trial}: {bad.size} tiles differ; first tile ({rows[b0]},{cols[b0]}) max {diff.max().item():.3e}; "
          f"cols of differing tiles {np.unique(cols[bad])[:12]}", flush=True)
