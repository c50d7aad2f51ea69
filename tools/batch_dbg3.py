import os, sys, time, threading, faulthandler
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2501_02483_b200 import api, workloads as W
from paper_2501_02483_b200._lib import lib, i32p
faulthandler.dump_traceback_later(110, exit=True)
lanes, P, conc = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
fam = W.InlaFamily()
ms = [fam.matrix(*t) for t in W.c5_thetas()[:P]]
opts = api.FactorOptions(tile_size=120, concurrent=conc)
import dataclasses
popts = dataclasses.replace(opts, concurrent=max(1, conc) if conc else 1)
pat = api._pattern_for(ms[0], popts if conc else dataclasses.replace(opts, concurrent=1))
def watch():
    time.sleep(60)
    for l in range(lanes):
        t = np.zeros(1, np.int32); n = np.zeros(1, np.int32)
        r = lib.tc_plan_debug_ticket(pat.plan.h, l, t.ctypes.data_as(i32p), n.ctypes.data_as(i32p))
        print("lane", l, "rc", r, "ticket", t[0], "of", n[0], flush=True)
threading.Thread(target=watch, daemon=True).start()
for it in range(3):
    t0 = time.perf_counter()
    out = api.logdet_many(ms, opts, lanes=lanes)
    print("call", it, time.perf_counter() - t0, flush=True)
