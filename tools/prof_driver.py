"""Minimal driver for ncu: set up a workload plan and run `--reps` factorisations."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2501_02483_b200 import api  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c2")
ap.add_argument("--tile", type=int, default=120)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--executor", default="persistent")
ap.add_argument("--ordering", default="auto")
a = ap.parse_args()
m = bench.build_matrix(a.workload)
opts = api.FactorOptions(tile_size=a.tile, executor=a.executor, ordering=a.ordering)
pat = api._pattern_for(m, opts)
plan = pat.plan
vals = torch.from_numpy(np.ascontiguousarray(pat.permuted_values(m))).cuda()
st = plan.new_storage()
sh = torch.cuda.current_stream().cuda_stream
for _ in range(a.reps):
    plan.pack(vals, pat.offsets(), st, sh)
    plan.factorize_async(st, 0, sh)
f, ld = plan.collect(0, sh)
print("fail", f, "logdet", ld, plan.info())
