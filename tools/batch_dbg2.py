import os, sys, time, faulthandler
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2501_02483_b200 import api, workloads as W
faulthandler.dump_traceback_later(100, exit=True)
fam = W.InlaFamily()
th = W.c5_thetas()[:6]
ms = [fam.matrix(*t) for t in th]
opts = api.FactorOptions(tile_size=120)
solo = np.array([api.logdet(api.factorize(m, opts)) for m in ms])
print("solo", solo)
for L in (1, 2, 3):
    out = api.logdet_many(ms, opts, lanes=L)
    print("logdet_many lanes", L, out - solo, flush=True)
fm = api.factorize_many(ms, opts, lanes=2)
print("factorize_many lanes 2", np.array([api.logdet(c) for c in fm]) - solo, flush=True)
