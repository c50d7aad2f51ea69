"""Persistent-executor task trace (legacy column-step breakdown: POTRF, TRSM, LAST per column).

    python tools/trace.py --workload c2 --tile 120 [--out gpurun_out/trace.npz]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2501_02483_b200 import api  # noqa: E402
from paper_2501_02483_b200._lib import check, lib, i32p, i64p  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c2")
ap.add_argument("--tile", type=int, default=120)
ap.add_argument("--ordering", default="auto")
ap.add_argument("--occupancy", type=int, default=0)
ap.add_argument("--lookahead", type=int, default=None)
ap.add_argument("--out", default="")
a = ap.parse_args()
m = bench.build_matrix(a.workload)
kw = {} if a.lookahead is None else {"lookahead": a.lookahead}
opts = api.FactorOptions(tile_size=a.tile, ordering=a.ordering, occupancy=a.occupancy, **kw)
pat = api._pattern_for(m, opts)
plan = pat.plan
vals = torch.from_numpy(np.ascontiguousarray(pat.permuted_values(m))).cuda()
st = plan.new_storage()
sh = torch.cuda.current_stream().cuda_stream
for _ in range(2):  # warm
    plan.pack(vals, pat.offsets(), st, sh)
    plan.factorize_async(st, 0, sh)
plan.collect(0, sh)
nt_, nl_ = np.zeros(1, np.int64), np.zeros(1, np.int64)
check("trace", lib.tc_plan_trace(plan.h, st.data_ptr(), sh, 0, None, None, 0, None,
                                  nt_.ctypes.data_as(i64p), nl_.ctypes.data_as(i64p)))
NT, NL = int(nt_[0]), int(nl_[0])
tr = np.zeros((NT, 4), np.int64)
tl = np.zeros(NT, np.int32)
lm = np.zeros((NL, 3), np.int32)
plan.pack(vals, pat.offsets(), st, sh)
check("trace", lib.tc_plan_trace(plan.h, st.data_ptr(), sh, NT, tr.ctypes.data_as(i64p), tl.ctypes.data_as(i32p),
                                  NL, lm.ctypes.data_as(i32p), nt_.ctypes.data_as(i64p), nl_.ctypes.data_as(i64p)))
t0 = tr[:, 0].min()
tr = tr.astype(np.float64)
tr[:, :3] = (tr[:, :3] - t0) / 1e3  # us
if a.out:
    np.savez_compressed(a.out, trace=tr, launch=tl, meta=lm)
total = tr[:, 2].max()
print(f"{a.workload}@{a.tile}: {NT} tasks, {NL} launches, span {total:.1f} us, T={plan.T}")
names = {0: "bulk", 1: "last", 2: "potrf", 3: "trsm", 4: "combine", 5: "logdet", 6: "splitk"}
cls = lm[tl, 2]
busy = (tr[:, 2] - tr[:, 1])
wait = (tr[:, 1] - tr[:, 0])
for c in sorted(set(cls.tolist())):
    sel = cls == c
    print(f"  {names[c]:8s} tasks {sel.sum():7d}  mean dur {busy[sel].mean():7.2f} us  sum {busy[sel].sum()/1e3:8.2f} ms"
          f"  mean dep-wait {wait[sel].mean():7.2f} us")
nsm = int(tr[:, 3].max()) + 1
print(f"  CTA-time busy fraction: {busy.sum() / (total * len(set(zip(tr[:,3].astype(int).tolist()))) * 1):.3f} (per SM id)")
# per-column critical path: POTRF(k) start/end, TRSM(k) end, LAST(k+1) start/end
T = plan.T
pot_s = np.full(T, np.nan); pot_e = np.full(T, np.nan)
trs_s = np.full(T, np.nan); trs_e = np.full(T, np.nan)
last_s = np.full(T, np.nan); last_e = np.full(T, np.nan)
kk = lm[tl, 1]
for c, s_arr, e_arr in ((2, pot_s, pot_e), (3, trs_s, trs_e), (1, last_s, last_e)):
    sel = np.where(cls == c)[0]
    for k in np.unique(kk[sel]):
        idx = sel[kk[sel] == k]
        s_arr[k] = tr[idx, 1].min()
        e_arr[k] = tr[idx, 2].max()
lo, hi = T // 4, 3 * T // 4
step = np.diff(pot_s)[lo:hi]
print(f"  column step (POTRF start to next POTRF start), middle half: mean {np.nanmean(step):.2f} us, "
      f"median {np.nanmedian(step):.2f}")
print(f"    POTRF duration        {np.nanmean((pot_e - pot_s)[lo:hi]):7.2f} us")
print(f"    POTRF end -> TRSM end {np.nanmean((trs_e - pot_e)[lo:hi]):7.2f} us")
print(f"    TRSM end -> LAST(k+1) start {np.nanmean((last_s[1:] - trs_e[:-1])[lo:hi]):7.2f} us")
print(f"    LAST(k+1) duration    {np.nanmean((last_e - last_s)[lo:hi]):7.2f} us")
print(f"    LAST end -> POTRF start {np.nanmean((pot_s - last_e)[lo:hi]):7.2f} us")
