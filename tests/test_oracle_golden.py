"""Pin the CPU oracle against the live-reference golden fixtures."""
import numpy as np
import pytest

import oracle as O
from conftest import CASE_NAMES, load_case, load_kats


@pytest.mark.parametrize("name", CASE_NAMES)
def test_oracle_integer_path_bit_exact(name):
    z = load_case(name)
    n, b, t, nt = int(z["n"]), int(z["b"]), int(z["t"]), int(z["nt"])
    bd = bool(z["bd"])
    if name != "e2000s":  # scrambled case is generated then permuted
        cp, ri, v = O.arrowhead(n, b, t, bd, seed=0)
        assert np.array_equal(cp, z["cp"]) and np.array_equal(ri, z["ri"])
        assert np.array_equal(v, z["vals"])  # bitwise, incl. diagonal sums
        assert O.arrowhead_nnz(n, b, t, bd) == int(z["nnz_closed"]) == cp[-1]
    cp, ri, v = z["cp"], z["ri"], z["vals"]
    bw, th, dens = O.structure(n, cp, ri)
    assert [bw, th] == list(z["stats"]) and dens == float(z["density"])
    assert np.array_equal(O.rcm_forward(n, cp, ri, th), z["rcm"])
    assert np.array_equal(O.rcm_forward(n, cp, ri, 0), z["rcm_full"])
    assert np.array_equal(O.nd_forward(n, bw, th), z["nd"])
    fills = [O.fill_count(n, cp, ri, f) for f in (None, z["rcm"], z["nd"])]
    assert fills == list(z["fill"])
    sel, _ = O.choose_ordering(n, cp, ri, [z["rcm"], z["nd"]])
    assert np.array_equal(sel, z["sel"])
    if "mindeg" in z:
        assert np.array_equal(O.min_degree_forward(n, cp, ri), z["mindeg"])
    pcp, pri, pv = O.permute(n, cp, ri, v, sel)
    assert np.array_equal(pcp, z["pcp"]) and np.array_equal(pri, z["pri"])
    assert np.array_equal(pv, z["pvals"])
    gr, gc, _ = O.tile_grid_of(n, nt, pcp, pri)
    assert np.array_equal(gr, z["g_rows"]) and np.array_equal(gc, z["g_cols"])
    fr, fc, fsm, acc = O.tile_symbolic(n, nt, gr, gc)
    assert np.array_equal(fr, z["f_rows"]) and np.array_equal(fc, z["f_cols"])
    assert np.array_equal(acc, z["accum"])
    T = fsm.shape[0]
    ts = O.task_stream(T, fsm)
    for k in ("type", "m", "k", "n", "target"):
        assert np.array_equal(ts[k], z["t_" + k]), k
    assert list(O.dag_levels(T, fsm, ts)) == list(z["dag"][:2])
    for w in (2, 4):
        plan = O.tree_plan(acc, w)
        assert sorted(plan) == list(z[f"plan{w}_slots"])
        for i, s in enumerate(sorted(plan)):
            assert np.array_equal(np.array(plan[s]), z[f"plan{w}_ranges"][i])
        assert np.array_equal(np.array(O.combine_steps(w)).reshape(-1, 2),
                              z[f"plan{w}_combine"].reshape(-1, 2))
    st = O.pack(n, nt, pcp, pri, pv, fsm, fr.size)
    assert np.array_equal(st, z["packed"])


@pytest.mark.parametrize("name", CASE_NAMES)
def test_oracle_numerics_match_reference(name):
    z = load_case(name)
    n, nt = int(z["n"]), int(z["nt"])
    fr, fc, fsm, acc = O.tile_symbolic(n, nt, z["g_rows"], z["g_cols"])
    ts = O.task_stream(fsm.shape[0], fsm)
    op, dst, s1, s2, _ = O.compile_ops(ts, fsm, fr.size)
    st = z["packed"].copy()
    p, info = O.run_ops(st, np.zeros((0, nt, nt)), op, dst, s1, s2, 0, op.size)
    assert info == -1
    # same engine (numba loops + BLAS dgemm) as the reference: bitwise here
    assert np.array_equal(st, z["factor"])
    r2 = O.replay_residual(st, z["packed"], op, dst, s1, s2, fr == fc)
    assert np.sqrt(r2 / z["anorm2"]) <= 1e-14
    assert abs(O.logdet(st, fsm, n, nt) - float(z["logdet"])) <= 1e-12 * max(1, abs(z["logdet"]))
    x = O.tile_solve(st, fsm, n, nt, z["rhs"], z["sel"])
    assert np.allclose(x, z["x"], rtol=0, atol=1e-12 * np.abs(z["x"]).max())
    # tree-reduction stream through the oracle executor
    plan = O.tree_plan(acc, 2)
    op2, d2, a2, b2, R = O.compile_ops(ts, fsm, fr.size, plan, 2)
    assert np.array_equal(np.stack([op2.astype(np.int64), d2, a2, b2]), z["ops_tree2"])
    st2 = z["packed"].copy()
    O.run_ops(st2, np.zeros((R, nt, nt)), op2, d2, a2, b2, 0, op2.size)
    assert np.array_equal(st2, z["factor_tree2"])


def test_oracle_kats():
    k = load_kats()
    a = k["potrf_in"].copy(order="F")
    assert O.potrf_t(a) == k["potrf_info"] == -1
    assert np.array_equal(a, k["potrf_out"])
    assert np.array_equal(a, [[2.0, 0.0], [1.0, 2.0]])
    x = k["trsm_b"].copy(order="F")
    assert O.trsm_t(k["trsm_l"].copy(order="F"), x) == -1
    assert np.array_equal(x, k["trsm_out"])
    c = k["syrk_c"].copy(order="F")
    O.syrk_t(k["syrk_a"].copy(order="F"), c)
    assert np.array_equal(c, k["syrk_out"])
    c = k["gemm_c"].copy(order="F")
    O.gemm_t(k["gemm_a"].copy(order="F"), k["gemm_b"].copy(order="F"), c)
    assert np.array_equal(c, k["gemm_out"])
    bad = np.array([[1.0, 2.0, 0.0], [2.0, 1.0, 0.0], [0.0, 0.0, 1.0]], order="F")
    assert O.potrf_t(bad) == k["potrf_bad_info"] == 1
    assert O.potrf_t(np.array([[np.nan, 0.0], [0.0, 1.0]], order="F")) == k["potrf_nan_info"] == -1
    assert O.trsm_t(np.array([[1.0, 0.0], [1.0, 0.0]], order="F"), np.ones((2, 2), order="F")) \
        == k["trsm_zero_info"] == 1
    cp, ri, v = O.canonical(30, k["coo_r"], k["coo_c"], k["coo_v"])
    assert np.array_equal(cp, k["coo_cp"]) and np.array_equal(ri, k["coo_ri"])
    assert np.array_equal(v, k["coo_vals"])


def test_oracle_dense6_dag():
    k = load_kats()
    r, c = np.tril_indices(6)
    fr, fc, fsm, acc = O.tile_symbolic(36, 6, r, c)
    ts = O.task_stream(6, fsm)
    counts = [int(np.sum(ts["type"] == x)) for x in (O.POTRF, O.SYRK, O.TRSM, O.GEMM)]
    assert counts == list(k["dense6_counts"]) == [6, 15, 15, 20]
    assert list(O.dag_levels(6, fsm, ts)) == list(k["dense6_cp_w"]) == [16, 15]
