"""Bitwise reproducibility of repeated factorisations (solo and concurrent lanes)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_2501_02483_b200 import api
name, nt, reps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
m = bench.build_matrix(name)
for occ in (1, 2):
    opts = api.FactorOptions(tile_size=nt, occupancy=occ)
    pat = api._pattern_for(m, opts)
    plan = pat.plan
    vals = torch.from_numpy(np.ascontiguousarray(pat.permuted_values(m))).cuda()
    st = plan.new_storage()
    sh = torch.cuda.current_stream().cuda_stream
    lds = []
    ref = None
    nbad = 0
    for r in range(reps):
        plan.pack(vals, pat.offsets(), st, sh)
        plan.factorize_async(st, 0, sh)
        f, ld = plan.collect(0, sh)
        lds.append(ld)
        if ref is None:
            ref = st.clone()
        elif not torch.equal(ref, st):
            nbad += 1
    print(f"{name}@{nt} occ{occ}: distinct logdets {len(set(lds))} of {reps}, storages differing {nbad}", flush=True)
