"""Fill-tile golden fixtures (tests/golden/make_golden_fill.py, live reference):
the tile elimination game (reference symbolic.py:98-123) on patterns whose
factor grid is strictly larger than the input grid, pinned bit-exactly for
the oracle and for the C++ host path, and the device factor against the
reference numba factor."""
import numpy as np
import pytest

import oracle as O
import oracle.workloads as OW
from conftest import load_case

FILL_CASES = ["i_inla", "j_vband"]
GEN = {
    "i_inla": lambda: (lambda f: (f.n, f.col_ptr, f.row_idx, f.values(0.5, 0.9, 1e-3)))(
        OW.InlaFamily(nx=10, ny=12, nsteps=20, nfix=3)),
    "j_vband": lambda: OW.c2(n=2400, t=24, seg_len=300, max_band=120, min_band=20),
}


@pytest.mark.parametrize("name", FILL_CASES)
def test_fill_oracle_bit_exact(name):
    z = load_case(name)
    n, nt = int(z["n"]), int(z["nt"])
    gn, cp, ri, v = GEN[name]()
    assert gn == n and np.array_equal(cp, z["cp"]) and np.array_equal(ri, z["ri"])
    assert np.array_equal(v, z["vals"])
    bw, th, _ = O.structure(n, cp, ri)
    assert [bw, th] == list(z["stats"])
    assert np.array_equal(O.rcm_forward(n, cp, ri, th), z["rcm"])
    assert np.array_equal(O.nd_forward(n, bw, th), z["nd"])
    assert [O.fill_count(n, cp, ri, f) for f in (None, z["rcm"], z["nd"])] == list(z["fill"])
    sel, _ = O.choose_ordering(n, cp, ri, [z["rcm"], z["nd"]])
    assert np.array_equal(sel, z["sel"])
    pcp, pri, pv = O.permute(n, cp, ri, v, sel)
    assert np.array_equal(pcp, z["pcp"]) and np.array_equal(pri, z["pri"]) and np.array_equal(pv, z["pvals"])
    gr, gc, _ = O.tile_grid_of(n, nt, pcp, pri)
    assert np.array_equal(gr, z["g_rows"]) and np.array_equal(gc, z["g_cols"])
    fr, fc, fsm, acc = O.tile_symbolic(n, nt, gr, gc)
    assert fr.size > gr.size  # genuinely exercises fill
    assert np.array_equal(fr, z["f_rows"]) and np.array_equal(fc, z["f_cols"])
    assert np.array_equal(acc, z["accum"])
    ts = O.task_stream(fsm.shape[0], fsm)
    for k in ("type", "m", "k", "n", "target"):
        assert np.array_equal(ts[k], z["t_" + k]), k
    for w in (2, 4):
        plan = O.tree_plan(acc, w)
        assert sorted(plan) == list(z[f"plan{w}_slots"])
    assert np.array_equal(O.pack(n, nt, pcp, pri, pv, fsm, fr.size), z["packed"])
    # the reference numba engine on the reconstructed op stream = the fixture factor
    op, dst, s1, s2, _ = O.compile_ops(ts, fsm, fr.size)
    st = z["packed"].copy()
    assert O.run_ops(st, np.zeros((0, nt, nt)), op, dst, s1, s2, 0, op.size) == (op.size, -1)
    assert np.array_equal(st, z["factor"])


@pytest.mark.parametrize("name", FILL_CASES)
def test_fill_host_cpp_bit_exact(name):
    """The C++ host path (tc_symbolic_*: etree-form elimination game, no T x T
    maps) on fill-producing patterns: factor grid, accum, task stream, op
    stream and tree plans equal the live reference."""
    from paper_2501_02483_b200 import ctsf, matcore, ordering, symbolic
    z = load_case(name)
    n, nt = int(z["n"]), int(z["nt"])
    m = matcore.SymmetricCsc(n, z["cp"], z["ri"], z["vals"])
    st = matcore.structure_stats(m)
    assert [st.bandwidth, st.thickness] == list(z["stats"])
    r = ordering.rcm(m, pinned_tail=st.thickness)
    nd = ordering.adaptable_nd(m, st)
    assert np.array_equal(r.forward, z["rcm"]) and np.array_equal(nd.forward, z["nd"])
    assert [ordering.symbolic_fill_count(m, p).nnz_factor for p in (None, r, nd)] == list(z["fill"])
    assert np.array_equal(ordering.select_ordering(m, [r, nd]).forward, z["sel"])
    pm = matcore.SymmetricCsc(n, z["pcp"], z["pri"], z["pvals"])
    g = ctsf.build_tile_grid(pm, nt)
    assert np.array_equal(g.tile_rows, z["g_rows"]) and np.array_equal(g.tile_cols, z["g_cols"])
    s = symbolic.tile_symbolic_factorize(g)
    fg = s.factor_grid
    assert np.array_equal(fg.tile_rows, z["f_rows"]) and np.array_equal(fg.tile_cols, z["f_cols"])
    assert np.array_equal(s.accum, z["accum"])
    tl = symbolic.enumerate_tasks(s)
    for k in ("type", "m", "k", "n", "target"):
        got = tl.task_type if k == "type" else getattr(tl, k)
        assert np.array_equal(got, z["t_" + k]), k
    for w in (2, 4):
        plan = symbolic.plan_tree_reduction(s, w)
        assert sorted(plan.chains) == list(z[f"plan{w}_slots"])
        for i, sl in enumerate(sorted(plan.chains)):
            assert np.array_equal(np.array(plan.chains[sl].ranges), z[f"plan{w}_ranges"][i])
    op, dst, s1, s2, _ = symbolic.compile_ops(s)
    fr, fc, fsm, acc = O.tile_symbolic(n, nt, z["g_rows"], z["g_cols"])
    o2 = O.compile_ops(O.task_stream(fsm.shape[0], fsm), fsm, fr.size)
    for a, b in zip((op, dst, s1, s2), o2[:4]):
        assert np.array_equal(a, b)
    assert np.array_equal(ctsf.pack_into_grid(pm, fg).storage, z["packed"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", FILL_CASES)
@pytest.mark.parametrize("executor", ["persistent", "graph"])
def test_fill_device_factor_vs_reference(name, executor):
    """api.factorize (device) on the fill cases vs the reference numba factor:
    factor <= 1e-12 relative Frobenius, backward error <= 1e-12, logdet vs
    the reference <= 1e-10, solve vs the reference tile solve <= 1e-10."""
    from paper_2501_02483_b200 import api, matcore
    z = load_case(name)
    n, nt = int(z["n"]), int(z["nt"])
    m = matcore.SymmetricCsc(n, z["cp"], z["ri"], z["vals"])
    ctx = api.factorize(m, api.FactorOptions(tile_size=nt, executor=executor))
    assert np.array_equal(ctx.permutation.forward, z["sel"])
    got = ctx.factor.host_storage()
    ref = z["factor"]
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-12
    from paper_2501_02483_b200.backend import impl
    fg = ctx.symbolic.factor_grid
    fr, fc, fsm, acc = O.tile_symbolic(n, nt, z["g_rows"], z["g_cols"])
    op, dst, s1, s2, _ = O.compile_ops(O.task_stream(fsm.shape[0], fsm), fsm, fr.size)
    e2 = impl.replay_residual(ctx.factor.storage, z["packed"], op, dst, s1, s2, fg.tile_rows == fg.tile_cols)
    assert np.sqrt(e2 / float(z["anorm2"])) <= 1e-12
    ld = api.logdet(ctx)
    assert abs(ld - float(z["logdet"])) <= 1e-10 * abs(float(z["logdet"]))
    x = api.solve(ctx, z["rhs"])
    assert np.linalg.norm(x - z["x"]) <= 1e-10 * np.linalg.norm(z["x"])


@pytest.mark.parametrize("name", FILL_CASES)
def test_expand_to_grid_and_unpack(name):
    """ctsf.expand_to_grid (reference ctsf.py:147-156): the input-grid packing
    re-homed into the (larger) factor grid equals packing straight into the
    factor grid (the reference fixture), extra fill slots stay zero, identity
    when the grids match, error when the target does not cover the source;
    unpack_to_csc (ctsf.py:159-184) round-trips the permuted matrix."""
    from paper_2501_02483_b200 import ctsf, matcore, symbolic
    z = load_case(name)
    n, nt = int(z["n"]), int(z["nt"])
    pm = matcore.SymmetricCsc(n, z["pcp"], z["pri"], z["pvals"])
    g = ctsf.build_tile_grid(pm, nt)
    fg = symbolic.tile_symbolic_factorize(g).factor_grid
    t_in = ctsf.pack_into_grid(pm, g)
    t_f = ctsf.expand_to_grid(t_in, fg)
    assert np.array_equal(t_f.storage, z["packed"])
    fill = fg.slots_of(np.setdiff1d(fg.keys, g.keys) % fg.tiles_per_side,
                       np.setdiff1d(fg.keys, g.keys) // fg.tiles_per_side)
    assert fill.size == fg.n_tiles - g.n_tiles and np.all(t_f.storage[fill] == 0.0)
    assert ctsf.expand_to_grid(t_f, fg) is t_f
    with pytest.raises(ValueError):
        ctsf.expand_to_grid(t_f, g)
    back = ctsf.unpack_to_csc(t_f)
    assert np.array_equal(back.col_ptr, pm.col_ptr) and np.array_equal(back.row_idx, pm.row_idx)
    assert np.array_equal(back.values, pm.values)
