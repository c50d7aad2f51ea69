import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2501_02483_b200 import api, workloads as W
m = W.InlaFamily(nx=10, ny=12, nsteps=20, nfix=3).matrix(0.5, 0.9, 1e-3)
occ = int(sys.argv[1]); nt = int(sys.argv[2])
opts = api.FactorOptions(tile_size=nt, ordering="identity", occupancy=occ)
pat = api._pattern_for(m, opts)
plan = pat.plan
vals = torch.from_numpy(np.ascontiguousarray(pat.permuted_values(m))).cuda()
st = plan.new_storage()
sh = torch.cuda.current_stream().cuda_stream
plan.pack(vals, pat.offsets(), st, sh)
plan.factorize_async(st, 0, sh)
f, ld = plan.collect(0, sh)
print("fail", f, "ld", ld)
np.save(sys.argv[3], st.cpu().numpy())
