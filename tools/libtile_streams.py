"""Same-box GPU baseline in the style of the paper's GPU prototype with its
per-worker streams ("each core is assigned its own CUDA stream";
SURVEY 8(f) #4): the reference op stream (POTRF/TRSM/SYRK/
GEMM per tile, reference symbolic.py:126-164 order) executed with library
kernels -- cuSOLVER potrf (torch.linalg.cholesky_ex), cuBLAS trsm
(solve_triangular) and gemm/syrk (addmm) -- one launch per tile op, ops owned
by the stream of their target tile column (W "workers"), cross-stream
read-after-write dependencies through CUDA events, the whole schedule captured
in one CUDA graph (so the number is library-kernel + dependency time, not
Python overhead).

    python tools/libtile_streams.py --workload c2 --tile 128 --streams 1,8,32 [--out f.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2501_02483_b200 import api, ctsf, symbolic  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c2")
ap.add_argument("--tile", type=int, default=128)
ap.add_argument("--streams", default="1,4,8,16,32")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--out", default="")
a = ap.parse_args()
m = bench.build_matrix(a.workload)
nt = a.tile
g = ctsf.build_tile_grid(m, nt)
s = symbolic.tile_symbolic_factorize(g)
op, dst, s1, s2 = [np.asarray(x) for x in symbolic.compile_ops(s)[:4]]
fg = s.factor_grid
fcol = np.asarray(fg.tile_cols)
tpl = torch.from_numpy(ctsf.pack_into_grid(m, fg).storage).cuda()
st = tpl.clone()
T = [st[i].T for i in range(st.shape[0])]  # column-major tile views (nt x nt)

# our executor on the same pattern, for the record
opts = api.FactorOptions(tile_size=nt, ordering="identity")
ctx = api.factorize(m, opts)
ours = ctx.factor.host_storage()


def schedule(W, streams):
    cur = torch.cuda.current_stream()
    for sm in streams:
        sm.wait_stream(cur)
    ready = {}  # slot -> (event, stream) of its final producer (POTRF / TRSM)
    for p in range(op.size):
        t, d = int(op[p]), int(dst[p])
        w = int(fcol[d]) % W
        sm = streams[w]
        with torch.cuda.stream(sm):
            for src in ((int(s1[p]),) if t == 3 else (int(s1[p]), int(s2[p])) if t in (2, 4) else ()):
                r = ready.get(src)
                if r is not None and r[1] != w:
                    sm.wait_event(r[0])
            D = T[d]
            if t == 1:  # POTRF
                L, _ = torch.linalg.cholesky_ex(D)
                D.copy_(L)
            elif t == 2:  # SYRK  C -= A A^T
                A = T[int(s1[p])]
                D.addmm_(A, A.T, alpha=-1.0)
            elif t == 3:  # TRSM  X L^T = B
                D.copy_(torch.linalg.solve_triangular(T[int(s1[p])].T, D, upper=True, left=False))
            elif t == 4:  # GEMM  C -= B A^T, src1 = A = L(k,n), src2 = B = L(m,n)
                D.addmm_(T[int(s2[p])], T[int(s1[p])].T, alpha=-1.0)
            if t in (1, 3):
                ev = torch.cuda.Event()
                ev.record(sm)
                ready[d] = (ev, w)
    for sm in streams:
        cur.wait_stream(sm)


res = {"workload": a.workload, "tile": nt, "ops": int(op.size), "tiles": int(st.shape[0]), "runs": []}
for W in [int(x) for x in a.streams.split(",")]:
    streams = [torch.cuda.Stream() for _ in range(W)]
    st.copy_(tpl)
    schedule(W, streams)  # warm (library handles, workspaces)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    st.copy_(tpl)
    torch.cuda.synchronize()
    with torch.cuda.graph(gr):
        schedule(W, streams)
    ts = []
    for _ in range(a.reps):
        st.copy_(tpl)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gr.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    got = st.cpu().numpy()
    rel = float(np.linalg.norm(got - ours) / np.linalg.norm(ours))
    res["runs"].append({"streams": W, "ms": min(ts), "all_ms": ts, "factor_rel_diff_vs_ours": rel})
    print(f"{a.workload}@{nt}: {op.size} library launches on {W} streams (graph): {min(ts):9.2f} ms  "
          f"(factor vs ours {rel:.1e})", flush=True)
    del gr
print(json.dumps(res))
if a.out:
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
