"""A/B of persistent-scheduler plan options on one workload (GPU box).

    python tools/ab_sched.py --workload c4 --tile 120 --variants default,nochain,nosplit,neither
Prints ms per factorisation (CUDA events, pack + factorise) and the logdet.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dataclasses  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2501_02483_b200 import api  # noqa: E402
from paper_2501_02483_b200.scheduler import DevicePlan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c4")
ap.add_argument("--tile", type=int, default=120)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--variants", default="default,nochain,nosplit,neither")
a = ap.parse_args()
m = bench.build_matrix(a.workload)
opts = api.FactorOptions(tile_size=a.tile, ordering="identity")
pat = api._pattern_for(m, opts)
vals = torch.from_numpy(np.ascontiguousarray(pat.permuted_values(m))).cuda()
base = pat.plan.options
VAR = {
    "default": {},
    "la1": {"lookahead": 1},
    "la3": {"lookahead": 3},
    "la4": {"lookahead": 4},
    "la6": {"lookahead": 6},
    "la8": {"lookahead": 8},
    "la10": {"lookahead": 10},
    "la12": {"lookahead": 12},
    "la16": {"lookahead": 16},
    "graph": {"executor": "graph"},
    "direct": {"executor": "direct"},
    "la2": {"lookahead": 2},
    "occ2": {"occupancy": 2},
    "occ2la2": {"occupancy": 2, "lookahead": 2},
    "occ2la4": {"occupancy": 2, "lookahead": 4},
}
st = pat.plan.new_storage()
sh = torch.cuda.current_stream().cuda_stream
for v in a.variants.split(","):
    popts = dataclasses.replace(base, **VAR[v])
    plan = DevicePlan(pat.symbolic.factor_grid, popts)
    off = pat.offsets()
    ts, lds = [], []
    for r in range(a.reps + 1):
        plan.pack(vals, off, st, sh)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.factorize_async(st, 0, sh)
        e1.record()
        f, ld = plan.collect(0, sh)
        torch.cuda.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1))
        lds.append(ld)
    print(f"{a.workload}@{a.tile} {v:8s} ms {min(ts):9.2f} (all {['%.1f' % t for t in ts]}) "
          f"logdet {lds[0]!r} same={len(set(lds)) == 1} fail={f}", flush=True)
    del plan
