"""Single factorisation, persistent grid reduced via `concurrent`: compare storages bitwise."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2501_02483_b200 import api, workloads as W
fam = W.InlaFamily()
m = fam.matrix(*W.c5_thetas()[int(sys.argv[1]) if len(sys.argv) > 1 else 0])
def run(conc, reps, occ=0):
    opts = api.FactorOptions(tile_size=120, concurrent=conc, occupancy=occ)
    pat = api._pattern_for(m, opts)
    plan = pat.plan
    vals = torch.from_numpy(np.ascontiguousarray(pat.permuted_values(m))).cuda()
    st = plan.new_storage()
    sh = torch.cuda.current_stream().cuda_stream
    outs = []
    for _ in range(reps):
        plan.pack(vals, pat.offsets(), st, sh)
        plan.factorize_async(st, 0, sh)
        f, ld = plan.collect(0, sh)
        outs.append(st.clone())
    return outs, pat
ref, pat = run(1, 1)
fg = pat.symbolic.factor_grid
for conc in (2, 4, 8):
    outs, _ = run(conc, 4)
    for i, o in enumerate(outs):
        d = (o - ref[0]).abs().amax(dim=(1, 2))
        bad = torch.nonzero(d > 0).flatten().cpu().numpy()
        if bad.size:
            s0 = int(bad[0])
            print(f"conc {conc} rep {i}: {bad.size} tiles differ; first slot {s0} tile ({fg.tile_rows[s0]},{fg.tile_cols[s0]}) max {d[s0].item():.2e}", flush=True)
        else:
            print(f"conc {conc} rep {i}: identical", flush=True)
