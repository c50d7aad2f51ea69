"""Generate golden fixtures from the LIVE reference (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Imports the reference ``tilechol`` package (pure Python + numba) from
``/root/reference/pkg/src`` and records, for a set of small/medium cases,
every integer artefact of the path (stats, orderings, fill counts, tile grid,
symbolic factor, task stream, tree plans, DAG stats) and the FP64 artefacts of
its numba backend (factor tiles from ``backend.impl.run_ops``, replay
residual, logdet, tile solve).  The op stream fed to the reference executor is
the reconstructed compiler (survey §8(c)); the reference ships no scheduler.
Fixtures land in ``tests/golden/*.npz`` and are committed; nothing at test
time reads /root/reference.
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

import oracle  # noqa: E402  (only for the op compiler reconstruction + solve)

CASES = [
    # name, n, b, t, block_diagonal, nt, scramble
    ("a64", 64, 4, 4, False, 8, False),
    ("b200", 200, 10, 6, False, 16, False),
    ("c500bd", 500, 20, 8, True, 40, False),
    ("d1000", 1000, 40, 10, False, 48, False),
    ("e2000s", 2000, 30, 10, False, 40, True),
    ("f48", 48, 40, 4, False, 8, False),
    ("g7", 7, 0, 0, False, 3, False),
    ("h1", 1, 0, 0, False, 4, False),
]


def scramble(m, seed=7):
    rng = np.random.default_rng(seed)
    t = matcore.structure_stats(m).thickness
    head = rng.permutation(m.n - t)
    fwd = np.concatenate([head, np.arange(m.n - t, m.n)]).astype(np.int64)
    return matcore.permute_symmetric(m, ordering.Permutation.from_forward(fwd))


def one(name, n, b, t, bd, nt, scr):
    spec = matcore.ArrowheadSpec(n=n, b=b, t=t, block_diagonal=bd, seed=0)
    m = matcore.generate_arrowhead(spec)
    if scr:
        m = scramble(m)
    out = {"n": n, "b": b, "t": t, "bd": int(bd), "nt": nt,
           "cp": m.col_ptr, "ri": m.row_idx, "vals": m.values,
           "nnz_closed": matcore.pattern_nnz_lower(spec)}
    st = matcore.structure_stats(m)
    out["stats"] = np.array([st.bandwidth, st.thickness])
    out["density"] = st.density_percent
    rcm = ordering.rcm(m, pinned_tail=st.thickness)
    rcm_full = ordering.rcm(m, pinned_tail=0)
    nd = ordering.adaptable_nd(m, st)
    out["rcm"] = rcm.forward
    out["rcm_full"] = rcm_full.forward
    out["nd"] = nd.forward
    out["fill"] = np.array([ordering.symbolic_fill_count(m, p).nnz_factor
                            for p in (ordering.Permutation.identity(n), rcm, nd)])
    sel = ordering.select_ordering(m, [rcm, nd])
    out["sel"] = sel.forward
    if n <= 64:
        out["mindeg"] = ordering.min_degree(m).forward
    pm = matcore.permute_symmetric(m, sel)
    out["pcp"], out["pri"], out["pvals"] = pm.col_ptr, pm.row_idx, pm.values
    g = ctsf.build_tile_grid(pm, nt)
    out["g_rows"], out["g_cols"] = g.tile_rows, g.tile_cols
    s = symbolic.tile_symbolic_factorize(g)
    fg = s.factor_grid
    out["f_rows"], out["f_cols"], out["accum"] = fg.tile_rows, fg.tile_cols, s.accum
    tl = symbolic.enumerate_tasks(s)
    out["t_type"], out["t_m"], out["t_k"], out["t_n"], out["t_target"] = (
        tl.task_type, tl.m, tl.k, tl.n, tl.target)
    ds = symbolic.dag_stats(s)
    out["dag"] = np.array([ds.critical_path, ds.max_width, ds.total_tasks])
    for w in (2, 4):
        plan = symbolic.plan_tree_reduction(s, w)
        slots = sorted(plan.chains)
        out[f"plan{w}_slots"] = np.array(slots, dtype=np.int64)
        out[f"plan{w}_ranges"] = np.array([plan.chains[x].ranges for x in slots],
                                          dtype=np.int64).reshape(len(slots), w, 2)
        out[f"plan{w}_combine"] = np.array(symbolic._combine_steps(w), dtype=np.int64)
    tm = ctsf.pack_into_grid(pm, fg)
    out["packed"] = tm.storage
    tasks = {"type": tl.task_type, "m": tl.m, "k": tl.k, "n": tl.n, "target": tl.target}
    S = fg.n_tiles
    op, dst, s1, s2, _ = oracle.compile_ops(tasks, fg.slot_map, S)
    fac = tm.storage.copy()
    p, info = backend.impl.run_ops(fac, np.zeros((0, nt, nt)), op, dst, s1, s2, 0, op.size)
    assert info == -1, (name, p, info)
    out["factor"] = fac
    diag = fg.tile_rows == fg.tile_cols
    err2 = backend.impl.replay_residual(fac, tm.storage, op, dst, s1, s2, diag)
    out["resid2"] = err2
    out["anorm2"] = float(np.sum(m.to_dense() ** 2)) if n <= 20000 else np.nan
    out["logdet"] = oracle.logdet(fac, fg.slot_map, n, nt)
    sgn, ld_dense = np.linalg.slogdet(m.to_dense())
    out["logdet_dense"] = ld_dense
    rhs = np.random.default_rng(3).standard_normal(n)
    out["rhs"] = rhs
    out["x"] = oracle.tile_solve(fac, fg.slot_map, n, nt, rhs, sel.forward)
    # tree-reduction path through the reference executor (W=2)
    plan = symbolic.plan_tree_reduction(s, 2)
    pl = {k: list(v.ranges) for k, v in plan.chains.items()}
    op2, dst2, s12, s22, R = oracle.compile_ops(tasks, fg.slot_map, S, pl, 2)
    fac2 = tm.storage.copy()
    p2, info2 = backend.impl.run_ops(fac2, np.zeros((max(R, 0), nt, nt)), op2, dst2, s12, s22, 0, op2.size)
    assert info2 == -1
    out["factor_tree2"] = fac2
    out["ops_tree2"] = np.stack([op2.astype(np.int64), dst2, s12, s22])
    np.savez_compressed(os.path.join(HERE, f"case_{name}.npz"), **out)
    print(name, "S", S, "P", tl.task_type.size, "resid", np.sqrt(err2 / out["anorm2"]))


def kats():
    imp = backend.impl
    out = {}
    a = np.array([[4.0, 2.0], [2.0, 5.0]])
    pa = a.copy(order="F")
    out["potrf_in"], out["potrf_info"] = a, imp.potrf_tile(pa)
    out["potrf_out"] = pa
    l = np.array([[2.0, 0.0], [1.0, 2.0]])
    x = np.array([[2.0, 3.0], [3.0, 5.0]])
    px = x.copy(order="F")
    out["trsm_l"], out["trsm_b"], out["trsm_info"] = l, x, imp.trsm_tile(l.copy(order="F"), px)
    out["trsm_out"] = px
    sa = np.array([[1.0, 2.0], [3.0, 4.0]])
    sc = np.array([[30.0, 0.0], [0.0, 30.0]])
    psc = sc.copy(order="F")
    imp.syrk_tile(sa.copy(order="F"), psc)
    out["syrk_a"], out["syrk_c"], out["syrk_out"] = sa, sc, psc
    ga = np.array([[1.0, 0.0], [0.0, 1.0]])
    gb = np.array([[2.0, 2.0], [0.0, 2.0]])
    gc = np.zeros((2, 2))
    pgc = gc.copy(order="F")
    imp.gemm_tile(ga.copy(order="F"), gb.copy(order="F"), pgc)
    out["gemm_a"], out["gemm_b"], out["gemm_c"], out["gemm_out"] = ga, gb, gc, pgc
    # failure semantics: non-positive pivot index, NaN passes, zero TRSM diag
    bad = np.array([[1.0, 2.0, 0.0], [2.0, 1.0, 0.0], [0.0, 0.0, 1.0]]).copy(order="F")
    out["potrf_bad_info"] = imp.potrf_tile(bad)
    nanm = np.array([[np.nan, 0.0], [0.0, 1.0]]).copy(order="F")
    out["potrf_nan_info"] = imp.potrf_tile(nanm)
    zl = np.array([[1.0, 0.0], [1.0, 0.0]]).copy(order="F")
    out["trsm_zero_info"] = imp.trsm_tile(zl, np.ones((2, 2), order="F"))
    # random KATs at nt=24 through the reference numba kernels
    rng = np.random.default_rng(11)
    nt = 24
    m0 = rng.standard_normal((nt, nt))
    spd = m0 @ m0.T + nt * np.eye(nt)
    pspd = spd.copy(order="F")
    out["rk_spd"], out["rk_potrf_info"] = spd, imp.potrf_tile(pspd)
    out["rk_potrf"] = pspd
    xb = rng.standard_normal((nt, nt))
    pxb = xb.copy(order="F")
    out["rk_trsm_b"], out["rk_trsm_info"] = xb, imp.trsm_tile(pspd, pxb)
    out["rk_trsm"] = pxb
    ca = rng.standard_normal((nt, nt))
    cb = rng.standard_normal((nt, nt))
    cc = rng.standard_normal((nt, nt))
    pc = cc.copy(order="F")
    imp.gemm_tile(ca.copy(order="F"), cb.copy(order="F"), pc)
    out["rk_ga"], out["rk_gb"], out["rk_gc"], out["rk_gemm"] = ca, cb, cc, pc
    pc2 = cc.copy(order="F")
    imp.syrk_tile(ca.copy(order="F"), pc2)
    out["rk_syrk"] = pc2
    # from_coordinates with duplicates (sum order semantics) and canonical errors
    n = 30
    rr = rng.integers(0, n, 400)
    cc_ = rng.integers(0, n, 400)
    vv = rng.standard_normal(400)
    rr = np.concatenate([rr, np.arange(n)])
    cc_ = np.concatenate([cc_, np.arange(n)])
    vv = np.concatenate([vv, np.full(n, 100.0)])
    m = matcore.from_coordinates(n, rr, cc_, vv, sum_duplicates=True)
    out["coo_r"], out["coo_c"], out["coo_v"] = rr, cc_, vv
    out["coo_cp"], out["coo_ri"], out["coo_vals"] = m.col_ptr, m.row_idx, m.values
    # dense 6x6 tile grid DAG
    g = ctsf.grid_from_tiles(36, 6, *np.tril_indices(6))
    s = symbolic.tile_symbolic_factorize(g)
    ds = symbolic.dag_stats(s)
    out["dense6_counts"] = np.array([ds.counts[k] for k in ("POTRF", "SYRK", "TRSM", "GEMM")])
    out["dense6_cp_w"] = np.array([ds.critical_path, ds.max_width])
    tt = symbolic.build_task_table(s, 2)
    out["dense6_owner2"] = np.array([tt.owner_of(int(r), int(c)) for r, c in
                                     zip(s.factor_grid.tile_rows, s.factor_grid.tile_cols)])
    np.savez_compressed(os.path.join(HERE, "kats.npz"), **out)
    print("kats ok")


if __name__ == "__main__":
    print("reference backend:", backend.BACKEND)
    kats()
    for c in CASES:
        one(*c)
