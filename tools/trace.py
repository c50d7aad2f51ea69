"""Persistent-executor task trace (GPU box): per-column critical-path breakdown.

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
if a.occupancy == 2:
    os.environ["TILECHOL_EXPERIMENTAL"] = "1"
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
# algorithmic flops per profiling class (serialised direct pass of the same plan)
from paper_2501_02483_b200._lib import f64p  # noqa: E402
pms, pcnt, pfl = np.zeros(7), np.zeros(7, np.int64), np.zeros(7)
plan.pack(vals, pat.offsets(), st, sh)
check("profile", lib.tc_plan_profile(plan.h, st.data_ptr(), sh, 7, pms.ctypes.data_as(f64p),
                                     pcnt.ctypes.data_as(i64p), pfl.ctypes.data_as(f64p)))
sm_peak = 37.15e12 / 148
cls = lm[tl, 2]
busy = (tr[:, 2] - tr[:, 1])
wait = (tr[:, 1] - tr[:, 0])
for c in sorted(set(cls.tolist())):
    sel = cls == c
    eff = pfl[c] / (busy[sel].sum() * 1e-6) / sm_peak if busy[sel].sum() > 0 else 0.0
    print(f"  {names[c]:8s} tasks {sel.sum():7d}  mean dur {busy[sel].mean():7.2f} us  sum {busy[sel].sum()/1e3:8.2f} ms"
          f"  mean dep-wait {wait[sel].mean():7.2f} us  gflop {pfl[c]/1e9:9.1f}  per-SM DMMA eff {eff:.3f}")
nsm = int(tr[:, 3].max()) + 1
ncta = len(np.unique(tr[:, 3]))
print(f"  CTA-time busy fraction: {busy.sum() / (total * ncta):.3f} over {ncta} SMs; dep-wait fraction "
      f"{wait.sum() / (total * ncta):.3f}")
# per-column critical path: POTRF(k), the critical TRSM of column k (chain),
# L_diag(k+1) (chain), M(k+1) and B(k+1)
T = plan.T
kind = lm[tl, 0] & 0xFF
chain = (lm[tl, 0] >> 8) & 1
mid = (lm[tl, 0] >> 9) & 1
sub = (lm[tl, 0] >> 10) & 1
kk = lm[tl, 1]


def span(sel):
    s_arr = np.full(T, np.nan)
    e_arr = np.full(T, np.nan)
    idx = np.nonzero(sel)[0]
    if idx.size:
        order = np.argsort(kk[idx], kind="stable")
        idx = idx[order]
        ks, starts = np.unique(kk[idx], return_index=True)
        for j, k in enumerate(ks):
            seg = idx[starts[j]:(starts[j + 1] if j + 1 < len(starts) else len(idx))]
            s_arr[k] = tr[seg, 1].min()
            e_arr[k] = tr[seg, 2].max()
    return s_arr, e_arr


pot_s, pot_e = span(cls == 2)
ct_s, ct_e = span((cls == 3) & (chain == 1) & (sub == 0))
c2_s, c2_e = span((cls == 3) & (chain == 1) & (sub == 1))
ld_s, ld_e = span((cls == 1) & (chain == 1) & (sub == 0))
lc_s, lc_e = span((cls == 1) & (chain == 1) & (sub == 1))
tr_s, tr_e = span((cls == 3) & (chain == 0))
lo_s, lo_e = span((cls == 1) & (chain == 0))
m_s, m_e = span((cls == 0) & (mid == 1))
b_s, b_e = span((cls == 0) & (mid == 0))
busy_all = tr[:, 2] - tr[:, 1]
for nm, sel in (("C1 TRSM", (cls == 3) & (chain == 1) & (sub == 0)), ("C2 TRSM", (cls == 3) & (chain == 1) & (sub == 1)),
                ("rest TRSM", (cls == 3) & (chain == 0)), ("L_diag", (cls == 1) & (chain == 1) & (sub == 0)),
                ("L_crit", (cls == 1) & (chain == 1) & (sub == 1)), ("L_off", (cls == 1) & (chain == 0)),
                ("near N", (cls == 0) & (mid == 1)), ("far B", (cls == 0) & (mid == 0))):
    if sel.any():
        print(f"    {nm:10s} tasks {sel.sum():8d} mean dur {busy_all[sel].mean():7.2f} us  p90 {np.percentile(busy_all[sel], 90):7.2f}"
              f"  mean wait {wait[sel].mean():7.2f}")
lo, hi = T // 4, 3 * T // 4
sl = slice(lo, hi)


def mean(x):
    return float(np.nanmean(x[sl]))


step = np.full(T, np.nan)
step[:-1] = np.diff(pot_s)
print(f"  column step (POTRF(k) start -> POTRF(k+1) start), middle half: mean {mean(step):.2f} us")
print(f"    POTRF(k) duration                      {mean(pot_e - pot_s):7.2f}")
nxt = lambda x: np.concatenate([x[1:], [np.nan]])  # noqa: E731  value at k+1
print(f"    POTRF(k) end -> crit TRSM(k) end       {mean(ct_e - pot_e):7.2f}")
print(f"    crit TRSM(k) end -> L_diag(k+1) start  {mean(nxt(ld_s) - ct_e):7.2f}")
print(f"    M(k+1) end - crit TRSM(k) end          {mean(nxt(m_e) - ct_e):7.2f}  (>0: M late)")
print(f"    B(k+1) end - crit TRSM(k) end          {mean(nxt(b_e) - ct_e):7.2f}  (>0: B late)")
print(f"    L_diag(k+1) duration                   {mean(ld_e - ld_s):7.2f}")
print(f"    L_crit(k+1) end - crit TRSM(k) end     {mean(nxt(lc_e) - ct_e):7.2f}   C1(k+1) start - POTRF(k+1) start "
      f"{mean(nxt(ct_s) - nxt(pot_s)):7.2f}")
print(f"    C2(k) end - POTRF(k) end               {mean(c2_e - pot_e):7.2f}   rest TRSM(k) end - POTRF(k) end "
      f"{mean(tr_e - pot_e):7.2f}   L_off(k+1) end - POTRF(k) end {mean(nxt(lo_e) - pot_e):7.2f}")
print(f"    L_diag(k+1) end -> POTRF(k+1) start    {mean(nxt(pot_s) - nxt(ld_e)):7.2f}")
print(f"    B(k) start - POTRF(k) start            {mean(b_s - pot_s):7.2f}   B(k) duration {mean(b_e - b_s):7.2f}")
# launch timeline around a middle column (relative to POTRF(kc) start, us)
kc = T // 2
t_ref = pot_s[kc]
lid = np.unique(tl)
l_s = np.full(NL, np.nan)
l_e = np.full(NL, np.nan)
l_n = np.zeros(NL, np.int64)
order_t = np.argsort(tl, kind="stable")
tls = tl[order_t]
bounds = np.searchsorted(tls, np.arange(NL + 1))
for L in range(NL):
    seg = order_t[bounds[L]:bounds[L + 1]]
    if seg.size:
        l_s[L] = tr[seg, 1].min()
        l_e[L] = tr[seg, 2].max()
        l_n[L] = seg.size
lk = lm[:, 1]
lkind = lm[:, 0] & 0xFF
lcls = lm[:, 2]
lchain = (lm[:, 0] >> 8) & 1
lmid = (lm[:, 0] >> 9) & 1
lsub = (lm[:, 0] >> 10) & 1
print(f"  launch timeline around column {kc} (us rel. to POTRF({kc}) start):")
for L in np.argsort(l_s):
    if np.isnan(l_s[L]) or lk[L] < kc - 1 or lk[L] > kc + 2:
        continue
    if l_e[L] - t_ref < -300 or l_s[L] - t_ref > 600:
        continue
    nm = {(0, 0): "B", (0, 1): "N"}.get((int(lcls[L]), int(lmid[L])), names.get(int(lcls[L]), "?"))
    if lcls[L] == 1:
        nm = "L_diag" if lchain[L] and not lsub[L] else ("L_crit" if lchain[L] else "L_off")
    if lcls[L] == 3:
        nm = "C1" if lchain[L] and not lsub[L] else ("C2" if lchain[L] else "TRSMr")
    print(f"    k={lk[L]:5d} {nm:7s} tasks {l_n[L]:4d}  start {l_s[L] - t_ref:9.1f}  end {l_e[L] - t_ref:9.1f}")
