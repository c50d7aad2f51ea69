"""Same-box GPU baseline in the style of the paper's GPU prototype (PAPER.md:388,
SURVEY 8(f) #4): the reference op stream (POTRF/TRSM/SYRK/GEMM per tile, in the
sequential left-looking order) executed with library kernels — cuSOLVER potrf
(torch.linalg.cholesky_ex), cuBLAS trsm (solve_triangular) and gemm (addmm) —
one launch per tile op on one stream, captured in a CUDA graph so the number
is library-kernel time, not Python overhead.

    python tools/libtile_baseline.py [--workload c2] [--tile 120]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2501_02483_b200 import api, ctsf, symbolic  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c2")
ap.add_argument("--tile", type=int, default=120)
a = ap.parse_args()
m = bench.build_matrix(a.workload)
nt = a.tile
g = ctsf.build_tile_grid(m, nt)
s = symbolic.tile_symbolic_factorize(g)
op, dst, s1, s2 = symbolic.compile_ops(s)[:4]
fg = s.factor_grid
tpl = torch.from_numpy(ctsf.pack_into_grid(m, fg).storage).cuda()
st = tpl.clone()
T = [st[i].T for i in range(st.shape[0])]  # column-major tile views (nt x nt)


def run():
    for p in range(op.size):
        t = int(op[p])
        d = T[int(dst[p])]
        if t == 1:  # POTRF
            L, _ = torch.linalg.cholesky_ex(d)
            d.copy_(L)
        elif t == 2:  # SYRK  C -= A A^T
            a_ = T[int(s1[p])]
            d.addmm_(a_, a_.T, alpha=-1.0)
        elif t == 3:  # TRSM  X L^T = B
            l_ = T[int(s1[p])]
            d.copy_(torch.linalg.solve_triangular(l_.T, d, upper=True, left=False))
        elif t == 4:  # GEMM  C -= B A^T, src1 = A = L(k,n), src2 = B = L(m,n)
            d.addmm_(T[int(s2[p])], T[int(s1[p])].T, alpha=-1.0)


st.copy_(tpl)
run()  # warm (library handles, workspaces)
torch.cuda.synchronize()
use_graph = True
try:
    gr = torch.cuda.CUDAGraph()
    st.copy_(tpl)
    with torch.cuda.graph(gr):
        run()
except Exception as e:  # noqa: BLE001
    print("graph capture failed, timing eager launches:", e)
    use_graph = False
ms = []
for _ in range(3):
    st.copy_(tpl)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if use_graph:
        gr.replay()
    else:
        run()
    e1.record()
    torch.cuda.synchronize()
    ms.append(e0.elapsed_time(e1))
ours = api.factorize(m, api.FactorOptions(tile_size=nt))
ref = ours.factor.host_storage()
rel = float(np.linalg.norm(st.cpu().numpy() - ref) / np.linalg.norm(ref))
print(f"{a.workload}@{nt}: per-tile cuSOLVER/cuBLAS op stream ({op.size} ops, "
      f"{'CUDA graph' if use_graph else 'eager'}): {min(ms):.1f} ms; factor rel diff vs ours {rel:.1e}")
