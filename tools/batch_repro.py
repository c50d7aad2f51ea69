"""Repeat the 64-problem INLA batch (lanes 4) and count bitwise mismatches across runs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2501_02483_b200 import api, workloads as W
fam = W.InlaFamily()
ms = [fam.matrix(*t) for t in W.c5_thetas()]
runs = int(sys.argv[1]) if len(sys.argv) > 1 else 4
lanes = int(sys.argv[2]) if len(sys.argv) > 2 else 4
ref = api.logdet_many(ms, api.FactorOptions(tile_size=120), lanes=1)
for r in range(runs):
    out = api.logdet_many(ms, api.FactorOptions(tile_size=120), lanes=lanes)
    bad = np.nonzero(out != ref)[0]
    print(f"run {r}: mismatches {bad.tolist()} max rel {np.max(np.abs(out - ref) / np.abs(ref)):.2e}", flush=True)
