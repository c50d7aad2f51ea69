"""Host-side (C++) preprocessing vs live-reference golden fixtures: bit-exact."""
import numpy as np
import pytest

import oracle as O
from conftest import CASE_NAMES, load_case
from paper_2501_02483_b200 import ctsf, matcore, ordering, symbolic
from paper_2501_02483_b200._backend_cuda import etree_fill_count


def _m(z, prefix=""):
    return matcore.SymmetricCsc(int(z["n"]), z[prefix + "cp"], z[prefix + "ri"], z[prefix + "vals"])


@pytest.mark.parametrize("name", CASE_NAMES)
def test_generator_and_stats(name):
    z = load_case(name)
    spec = matcore.ArrowheadSpec(int(z["n"]), int(z["b"]), int(z["t"]), bool(z["bd"]), seed=0)
    assert matcore.pattern_nnz_lower(spec) == int(z["nnz_closed"])
    if name != "e2000s":
        m = matcore.generate_arrowhead(spec)
        assert np.array_equal(m.col_ptr, z["cp"]) and np.array_equal(m.row_idx, z["ri"])
        assert np.array_equal(m.values, z["vals"])  # bitwise incl. diagonal sums
    m = _m(z)
    m.validate()
    st = matcore.structure_stats(m)
    assert [st.bandwidth, st.thickness] == list(z["stats"])
    assert st.density_percent == float(z["density"])


@pytest.mark.parametrize("name", CASE_NAMES)
def test_orderings_and_fill(name):
    z = load_case(name)
    m = _m(z)
    st = matcore.structure_stats(m)
    r = ordering.rcm(m, pinned_tail=st.thickness)
    assert np.array_equal(r.forward, z["rcm"])
    assert np.array_equal(ordering.rcm(m, 0).forward, z["rcm_full"])
    nd = ordering.adaptable_nd(m, st)
    assert np.array_equal(nd.forward, z["nd"])
    fills = [ordering.symbolic_fill_count(m, p).nnz_factor for p in (None, r, nd)]
    assert fills == list(z["fill"])
    sel = ordering.select_ordering(m, [r, nd])
    assert np.array_equal(sel.forward, z["sel"])
    if "mindeg" in z:
        assert np.array_equal(ordering.min_degree(m).forward, z["mindeg"])
    pm = matcore.permute_symmetric(m, sel)
    assert np.array_equal(pm.col_ptr, z["pcp"]) and np.array_equal(pm.row_idx, z["pri"])
    assert np.array_equal(pm.values, z["pvals"])


@pytest.mark.parametrize("name", CASE_NAMES)
def test_tile_symbolic_tasks_plans(name):
    z = load_case(name)
    n, nt = int(z["n"]), int(z["nt"])
    pm = _m(z, "p")
    g = ctsf.build_tile_grid(pm, nt)
    assert np.array_equal(g.tile_rows, z["g_rows"]) and np.array_equal(g.tile_cols, z["g_cols"])
    g2 = ctsf.grid_from_tiles(n, nt, z["g_rows"], z["g_cols"])
    assert np.array_equal(g2.tile_rows, z["g_rows"]) and np.array_equal(g2.tile_cols, z["g_cols"])
    for gg in (g, g2):
        s = symbolic.tile_symbolic_factorize(gg)
        fg = s.factor_grid
        assert np.array_equal(fg.tile_rows, z["f_rows"]) and np.array_equal(fg.tile_cols, z["f_cols"])
        assert np.array_equal(s.accum, z["accum"])
    tl = symbolic.enumerate_tasks(s)
    for k in ("type", "m", "k", "n", "target"):
        got = tl.task_type if k == "type" else getattr(tl, k)
        assert np.array_equal(got, z["t_" + k]), k
    ds = symbolic.dag_stats(s)
    assert [ds.critical_path, ds.max_width, ds.total_tasks] == list(z["dag"])
    for w in (2, 4):
        plan = symbolic.plan_tree_reduction(s, w)
        assert sorted(plan.chains) == list(z[f"plan{w}_slots"])
        for i, sl in enumerate(sorted(plan.chains)):
            assert np.array_equal(np.array(plan.chains[sl].ranges), z[f"plan{w}_ranges"][i])
            assert np.array_equal(np.array(plan.chains[sl].combine).reshape(-1, 2),
                                  z[f"plan{w}_combine"].reshape(-1, 2))
    # op compiler vs oracle reconstruction (sequential and tree W=2)
    fr, fc, fsm, acc = O.tile_symbolic(n, nt, z["g_rows"], z["g_cols"])
    ts = O.task_stream(fsm.shape[0], fsm)
    mine = symbolic.compile_ops(s, 0)
    ref = O.compile_ops(ts, fsm, fr.size)
    for a, b in zip(mine[:4], ref[:4]):
        assert np.array_equal(a, b)
    mine2 = symbolic.compile_ops(s, 2)
    assert np.array_equal(np.stack([mine2[0].astype(np.int64), mine2[1], mine2[2], mine2[3]]), z["ops_tree2"])
    # packing
    tm = ctsf.pack_into_grid(pm, fg)
    assert np.array_equal(tm.storage, z["packed"])
    back = ctsf.unpack_to_csc(ctsf.pack_into_grid(pm, g))
    assert np.array_equal(back.col_ptr, pm.col_ptr) and np.array_equal(back.values, pm.values)


def test_etree_fill_count_plugin():
    z = load_case("e2000s")
    n = int(z["n"])
    cols = np.repeat(np.arange(n), np.diff(z["cp"]))
    rr = z["ri"].astype(np.int64)
    off = rr != cols
    hi, lo = rr[off], cols[off]
    o = np.argsort(hi, kind="stable")
    ptr = np.zeros(n + 1, dtype=np.int64)
    ptr[1:] = np.cumsum(np.bincount(hi, minlength=n))
    assert etree_fill_count(n, ptr, lo[o]) + n == int(z["fill"][0])


def test_dense6_kat_and_threshold_boundaries():
    r, c = np.tril_indices(6)
    s = symbolic.tile_symbolic_factorize(ctsf.grid_from_tiles(36, 6, r, c))
    ds = symbolic.dag_stats(s)
    assert ds.counts == {"POTRF": 6, "SYRK": 15, "TRSM": 15, "GEMM": 20}
    assert (ds.critical_path, ds.max_width) == (16, 15)
    assert symbolic._combine_steps(3) == ((0, 1), (0, 2))
    assert symbolic._combine_steps(4) == ((0, 1), (2, 3), (0, 2))
    assert symbolic._combine_steps(5) == ((0, 1), (2, 3), (0, 2), (0, 4))
    # SPEC.md:600 threshold rule: chain length 2P-1 / 2P / 2P+1
    for P in (2, 3, 4):
        for L, want in ((2 * P - 1, False), (2 * P, True), (2 * P + 1, True)):
            n = L + 1
            rows = np.arange(n)
            cols = np.zeros(n, dtype=np.int64)
            g = ctsf.grid_from_tiles(n, 1, np.r_[np.full(n, n - 1), rows], np.r_[rows, cols])
            s = symbolic.tile_symbolic_factorize(g)
            plan = symbolic.plan_tree_reduction(s, P)
            last = s.factor_grid.slot(n - 1, n - 1)
            assert int(s.accum[last]) == L
            assert (last in plan.chains) == want


def test_from_coordinates_semantics():
    from conftest import load_kats
    k = load_kats()
    m = matcore.from_coordinates(30, k["coo_r"], k["coo_c"], k["coo_v"])
    assert np.array_equal(m.col_ptr, k["coo_cp"]) and np.array_equal(m.row_idx, k["coo_ri"])
    assert np.array_equal(m.values, k["coo_vals"])
    from paper_2501_02483_b200.errors import MatrixFormatError
    with pytest.raises(MatrixFormatError):
        matcore.from_coordinates(2, [0, 1, 1], [0, 1, 0], [1.0, 1.0, 1.0], sum_duplicates=False) \
            if False else matcore.from_coordinates(2, [0, 1, 1, 1], [0, 1, 0, 0], [1, 1, 1, 1.0], False)
    with pytest.raises(MatrixFormatError, match="missing diagonal entry in column 2"):
        matcore.from_coordinates(2, [0], [0], [1.0])
    with pytest.raises(MatrixFormatError, match="non-positive"):
        matcore.from_coordinates(2, [0, 1], [0, 1], [1.0, -1.0])


@pytest.mark.parametrize("name", CASE_NAMES)
def test_factor_column_counts_sum_to_fill(name):
    z = load_case(name)
    m = _m(z)
    for f, want in ((None, z["fill"][0]), (z["rcm"], z["fill"][1]), (z["nd"], z["fill"][2])):
        p = None if f is None else ordering.Permutation.from_forward(f)
        c = ordering.factor_column_counts(m, p)
        assert int(c.sum()) == int(want) and c.min() >= 1
    # against explicit dense symbolic elimination for the small cases
    if int(z["n"]) <= 200:
        n = int(z["n"])
        S = O.dense_of(n, z["cp"], z["ri"], np.ones_like(z["vals"])) != 0
        for k in range(n):
            below = k + 1 + np.flatnonzero(S[k + 1:, k])
            S[np.ix_(below, below)] = True
        assert np.array_equal(ordering.factor_column_counts(m), np.tril(S).sum(axis=0))


def test_inla_lincomb_is_bitwise_values():
    """Device value assembly contract: the family's (coef, basis) sequence
    evaluated left to right reproduces values(theta) bitwise."""
    from paper_2501_02483_b200 import workloads as W
    fam = W.InlaFamily(nx=6, ny=7, nsteps=5, nfix=2)
    for th in W.c5_thetas()[::7]:
        coef, basis = fam.lincomb(*th)
        assert len(coef) == len(basis) <= 16
        v = coef[0] * basis[0]
        for c, b in zip(coef[1:], basis[1:]):
            v = v + c * b
        assert np.array_equal(v, fam.values(*th))


def test_occupancy_and_concurrency_options_validated():
    """occupancy 1/2 and concurrent >= 1 are accepted (the round-1 race is
    fixed); anything else is rejected."""
    import pytest
    from paper_2501_02483_b200.api import FactorOptions
    FactorOptions(occupancy=1, concurrent=1)
    FactorOptions(occupancy=2, concurrent=4)
    with pytest.raises(ValueError):
        FactorOptions(occupancy=3)
    with pytest.raises(ValueError):
        FactorOptions(concurrent=0)


def test_select_ordering_zero_fill_short_circuit():
    """Zero-fill identity: lazy candidates are never evaluated and the result
    is identity, as the reference's eager policy returns (ordering.py:266-275)."""
    from paper_2501_02483_b200 import matcore, ordering
    m = matcore.generate_arrowhead(matcore.ArrowheadSpec(n=300, b=10, t=5, seed=0))
    called = []

    def cand():
        called.append(1)
        return ordering.Permutation.identity(m.n)
    p = ordering.select_ordering(m, [cand, cand])
    assert p.is_identity() and not called


def test_zero_fill_shortcut_matches_etree_count():
    """tc_zero_fill (parallel perfect-elimination test in front of the
    sequential elimination-tree count, ordering.select_ordering) agrees with
    the reference fill count: perfect <=> nnz(L) == nnz(lower A), and then
    offdiag + n == nnz(L).  Band+arrow (zero fill), variable band (fill)."""
    import numpy as np
    from paper_2501_02483_b200 import matcore, ordering
    from paper_2501_02483_b200._lib import lib, ptr, i64p, i32p
    cases = [matcore.generate_arrowhead(matcore.ArrowheadSpec(3000, 60, 20, seed=1)),
             matcore.generate_arrowhead(matcore.ArrowheadSpec(500, 7, 3, block_diagonal=True, seed=2))]
    m = cases[0]
    p = ordering.rcm(m, pinned_tail=0)
    cases.append(matcore.permute_symmetric(m, p))  # scrambled: fill appears
    for m in cases:
        cp, ri = ordering._csc(m)
        perfect, offd = np.zeros(1, dtype=np.int32), np.zeros(1, dtype=np.int64)
        assert lib.tc_zero_fill(m.n, ptr(cp, i64p), ptr(ri, i32p), ptr(perfect, i32p), ptr(offd, i64p)) == 0
        nnz_l = ordering.symbolic_fill_count(m, None).nnz_factor
        assert bool(perfect[0]) == (nnz_l == int(offd[0]) + m.n)
        if perfect[0]:
            assert int(offd[0]) + m.n == nnz_l
        else:
            assert nnz_l > int(offd[0]) + m.n
