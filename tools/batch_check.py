import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2501_02483_b200 import api, matcore, workloads as W
fam = W.InlaFamily()
th = W.c5_thetas()[:8]
ms = [fam.matrix(*t) for t in th]
solo_opts = api.FactorOptions(tile_size=120)
solo = np.array([api.logdet(api.factorize(m, solo_opts)) for m in ms])
for L in (1, 2, 4):
    out = api.logdet_many(ms, api.FactorOptions(tile_size=120), lanes=L)
    print("lanes", L, "max |diff|", np.abs(out - solo).max(), "equal", np.array_equal(out, solo), flush=True)
opts = api.FactorOptions(tile_size=120, concurrent=4)
pat = api._pattern_for(ms[0], opts)
plan = pat.plan
coef, basis = fam.lincomb(*th[0])
bd = torch.from_numpy(np.stack([pat.permuted_values(matcore.SymmetricCsc(ms[0].n, ms[0].col_ptr, ms[0].row_idx, b)) for b in basis])).cuda()
s1, s2 = plan.new_storage(), plan.new_storage()
sh = torch.cuda.current_stream().cuda_stream
plan.pack_lincomb(bd, coef, pat.offsets(), s1, sh)
plan.pack(torch.from_numpy(np.ascontiguousarray(pat.permuted_values(ms[0]))).cuda(), pat.offsets(), s2, sh)
torch.cuda.synchronize()
print("pack_lincomb == pack:", torch.equal(s1, s2), (s1 - s2).abs().max().item())
