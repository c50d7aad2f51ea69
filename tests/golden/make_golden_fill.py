"""Golden fixtures WITH FILL TILES from the LIVE reference (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_fill.py

The arrowhead cases of make_golden.py all have S_in == S_factor (no fill), so
they never exercise the tile elimination game (reference symbolic.py:98-123)
beyond the trivial case.  These two cases do:

* ``i_inla``  — a small INLA precision Q(theta) (App. A3 recipe on a 10 x 12
  grid, 20 time steps, 3 fixed effects; oracle/workloads.InlaFamily) at nt=40:
  the block-tridiagonal time coupling creates fill tiles;
* ``j_vband`` — a piecewise variable-band arrowhead (App. A2 recipe with 300-
  column segments, bands 20-120) at nt=24: band drops between segments create
  fill tiles.

The matrices are built by the oracle generators (numpy/scipy) and handed to
the reference as ``tilechol.matcore.SymmetricCsc``; every integer artefact and
the reference numba factor are recorded.  Nothing at test time reads
/root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

from tilechol import backend, ctsf, matcore, ordering, symbolic  # noqa: E402

import oracle  # noqa: E402
import oracle.workloads as OW  # noqa: E402

FILL_CASES = {
    "i_inla": dict(gen="inla", nt=40, args=dict(nx=10, ny=12, nsteps=20, nfix=3), theta=(0.5, 0.9, 1e-3)),
    "j_vband": dict(gen="vband", nt=24, args=dict(n=2400, t=24, seg_len=300, max_band=120, min_band=20)),
}


def build(spec):
    if spec["gen"] == "inla":
        f = OW.InlaFamily(**spec["args"])
        return f.n, f.col_ptr, f.row_idx, f.values(*spec["theta"])
    return OW.c2(**spec["args"])


def one(name, spec):
    n, cp, ri, vals = build(spec)
    nt = spec["nt"]
    m = matcore.SymmetricCsc(n, cp, ri, vals)
    m.validate()
    out = {"n": n, "nt": nt, "gen": spec["gen"], "cp": cp, "ri": ri, "vals": vals}
    st = matcore.structure_stats(m)
    out["stats"] = np.array([st.bandwidth, st.thickness])
    rcm = ordering.rcm(m, pinned_tail=st.thickness)
    nd = ordering.adaptable_nd(m, st)
    out["rcm"], out["nd"] = rcm.forward, nd.forward
    out["fill"] = np.array([ordering.symbolic_fill_count(m, p).nnz_factor
                            for p in (ordering.Permutation.identity(n), rcm, nd)])
    sel = ordering.select_ordering(m, [rcm, nd])
    out["sel"] = sel.forward
    pm = matcore.permute_symmetric(m, sel)
    out["pcp"], out["pri"], out["pvals"] = pm.col_ptr, pm.row_idx, pm.values
    g = ctsf.build_tile_grid(pm, nt)
    out["g_rows"], out["g_cols"] = g.tile_rows, g.tile_cols
    s = symbolic.tile_symbolic_factorize(g)
    fg = s.factor_grid
    out["f_rows"], out["f_cols"], out["accum"] = fg.tile_rows, fg.tile_cols, s.accum
    assert fg.n_tiles > g.n_tiles, (name, "expected fill tiles")
    tl = symbolic.enumerate_tasks(s)
    out["t_type"], out["t_m"], out["t_k"], out["t_n"], out["t_target"] = (
        tl.task_type, tl.m, tl.k, tl.n, tl.target)
    for w in (2, 4):
        plan = symbolic.plan_tree_reduction(s, w)
        slots = sorted(plan.chains)
        out[f"plan{w}_slots"] = np.array(slots, dtype=np.int64)
        out[f"plan{w}_ranges"] = np.array([plan.chains[x].ranges for x in slots],
                                          dtype=np.int64).reshape(len(slots), w, 2)
    tm = ctsf.pack_into_grid(pm, fg)
    out["packed"] = tm.storage
    tasks = {"type": tl.task_type, "m": tl.m, "k": tl.k, "n": tl.n, "target": tl.target}
    op, dst, s1, s2, _ = oracle.compile_ops(tasks, fg.slot_map, fg.n_tiles)
    fac = tm.storage.copy()
    p, info = backend.impl.run_ops(fac, np.zeros((0, nt, nt)), op, dst, s1, s2, 0, op.size)
    assert info == -1, (name, p, info)
    out["factor"] = fac
    diag = fg.tile_rows == fg.tile_cols
    out["resid2"] = backend.impl.replay_residual(fac, tm.storage, op, dst, s1, s2, diag)
    dense = m.to_dense()
    out["anorm2"] = float(np.sum(dense ** 2))
    out["logdet"] = oracle.logdet(fac, fg.slot_map, n, nt)
    out["logdet_dense"] = np.linalg.slogdet(dense)[1]
    rhs = np.random.default_rng(5).standard_normal(n)
    out["rhs"] = rhs
    out["x"] = oracle.tile_solve(fac, fg.slot_map, n, nt, rhs, sel.forward)
    np.savez_compressed(os.path.join(HERE, f"case_{name}.npz"), **out)
    print(name, "n", n, "S_in", g.n_tiles, "S_factor", fg.n_tiles, "P", tl.task_type.size,
          "resid", np.sqrt(out["resid2"] / out["anorm2"]))


if __name__ == "__main__":
    for nm, sp in FILL_CASES.items():
        one(nm, sp)
