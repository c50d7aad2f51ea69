import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2501_02483_b200 import api, workloads as W
fam = W.InlaFamily()
ms = [fam.matrix(*t) for t in W.c5_thetas()]
ref = api.logdet_many(ms, api.FactorOptions(tile_size=120), lanes=1)
for r in range(3):
    out = api.logdet_many(ms, api.FactorOptions(tile_size=120, concurrent=2), lanes=2)
    bad = np.nonzero(out != ref)[0]
    print(f"run {r}: mismatches {bad.tolist()} max rel {np.max(np.abs(out - ref) / np.abs(ref)):.2e}", flush=True)
