"""GPU parity: the sm_100a path vs the oracle / live-reference golden fixtures.

FP64 tolerances (north star): backward error ||PAP^T - LL^T||_F/||A||_F <= 1e-12,
logdet relative difference <= 1e-10, solve residual <= 1e-10; factors are
compared with the reference factor at <= 1e-12 relative Frobenius (the two
reference backends themselves differ by ~1e-16, never bitwise).
"""
import numpy as np
import pytest

import oracle as O
from conftest import CASE_NAMES, load_case, load_kats

pytestmark = pytest.mark.gpu

BACKWARD_TOL = 1e-12
LOGDET_TOL = 1e-10
SOLVE_TOL = 1e-10
FACTOR_TOL = 1e-12


@pytest.fixture(scope="module")
def torch():
    import torch as t
    assert t.cuda.is_available(), "gpu tests need a CUDA device"
    return t


def _imports():
    from paper_2501_02483_b200 import api, ctsf, matcore, symbolic
    from paper_2501_02483_b200.backend import impl
    return api, ctsf, matcore, symbolic, impl


def relf(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def anorm_f(cp, vals):
    d = vals[cp[:-1]]
    return float(np.sqrt(2.0 * np.sum(vals ** 2) - np.sum(d ** 2)))


# ------------------------------------------------------------- tile KATs --
def test_tile_kats(torch):
    *_, impl = _imports()
    k = load_kats()
    a = k["potrf_in"].copy(order="F")
    assert impl.potrf_tile(a) == -1
    assert np.array_equal(a, k["potrf_out"])
    x = k["trsm_b"].copy(order="F")
    assert impl.trsm_tile(k["trsm_l"].copy(order="F"), x) == -1
    assert np.allclose(x, k["trsm_out"], rtol=0, atol=1e-15)
    c = k["syrk_c"].copy(order="F")
    impl.syrk_tile(k["syrk_a"].copy(order="F"), c)
    assert np.array_equal(c, k["syrk_out"])
    c = k["gemm_c"].copy(order="F")
    impl.gemm_tile(k["gemm_a"].copy(order="F"), k["gemm_b"].copy(order="F"), c)
    assert np.array_equal(c, k["gemm_out"])
    bad = np.array([[1.0, 2.0, 0.0], [2.0, 1.0, 0.0], [0.0, 0.0, 1.0]], order="F")
    assert impl.potrf_tile(bad) == k["potrf_bad_info"] == 1
    assert impl.potrf_tile(np.array([[np.nan, 0.0], [0.0, 1.0]], order="F")) == -1
    assert impl.trsm_tile(np.array([[1.0, 0.0], [1.0, 0.0]], order="F"), np.ones((2, 2), order="F")) == 1
    # random nt=24 KATs from the reference numba kernels
    a = k["rk_spd"].copy(order="F")
    assert impl.potrf_tile(a) == -1
    assert relf(a, k["rk_potrf"]) < 1e-14
    x = k["rk_trsm_b"].copy(order="F")
    assert impl.trsm_tile(k["rk_potrf"].copy(order="F"), x) == -1
    assert relf(x, k["rk_trsm"]) < 1e-13
    c = k["rk_gc"].copy(order="F")
    impl.gemm_tile(k["rk_ga"].copy(order="F"), k["rk_gb"].copy(order="F"), c)
    assert relf(c, k["rk_gemm"]) < 1e-14
    c = k["rk_gc"].copy(order="F")
    impl.syrk_tile(k["rk_ga"].copy(order="F"), c)
    assert relf(c, k["rk_syrk"]) < 1e-14


@pytest.mark.parametrize("nt", [1, 3, 8, 17, 40, 48, 64, 120, 128, 160, 200, 240, 320, 480, 600])
def test_tile_kernels_vs_torch_fp64(torch, nt):
    """Each tile kernel vs a plain PyTorch fp64 reference of the same op."""
    *_, impl = _imports()
    g = torch.Generator().manual_seed(nt)
    m0 = torch.randn(nt, nt, generator=g, dtype=torch.float64)
    spd = m0 @ m0.T + nt * torch.eye(nt, dtype=torch.float64)
    L = torch.linalg.cholesky(spd)
    a = spd.numpy().copy(order="F")
    assert impl.potrf_tile(a) == -1
    assert relf(a, L.numpy()) < 1e-13
    assert np.all(np.triu(a, 1) == 0.0)
    b = torch.randn(nt, nt, generator=g, dtype=torch.float64)
    x = b.numpy().copy(order="F")
    assert impl.trsm_tile(L.numpy().copy(order="F"), x) == -1
    ref = torch.linalg.solve_triangular(L, b.T, upper=False).T
    assert relf(x, ref.numpy()) < 1e-12
    A = torch.randn(nt, nt, generator=g, dtype=torch.float64)
    B = torch.randn(nt, nt, generator=g, dtype=torch.float64)
    Cm = torch.randn(nt, nt, generator=g, dtype=torch.float64)
    c = Cm.numpy().copy(order="F")
    impl.gemm_tile(A.numpy().copy(order="F"), B.numpy().copy(order="F"), c)
    assert relf(c, (Cm - B @ A.T).numpy()) < 1e-13
    c = Cm.numpy().copy(order="F")
    impl.syrk_tile(A.numpy().copy(order="F"), c)
    assert relf(c, (Cm - A @ A.T).numpy()) < 1e-13
    c = Cm.numpy().copy(order="F")
    impl.geadd_tile(A.numpy().copy(order="F"), c)
    assert np.array_equal(c, (Cm + A).numpy())
    # device tensors operated on in place (storage[s].T views)
    st = torch.stack([spd.T.contiguous(), b.T.contiguous()]).cuda()
    assert impl.potrf_tile(st[0].T) == -1
    assert relf(st[0].T.cpu().numpy(), L.numpy()) < 1e-13


# ------------------------------------------------ plugin seam: run_ops --
@pytest.mark.parametrize("name", CASE_NAMES)
def test_run_ops_matches_reference(torch, name):
    api, ctsf, matcore, symbolic, impl = _imports()
    z = load_case(name)
    n, nt = int(z["n"]), int(z["nt"])
    fr, fc, fsm, acc = O.tile_symbolic(n, nt, z["g_rows"], z["g_cols"])
    ts = O.task_stream(fsm.shape[0], fsm)
    op, dst, s1, s2, _ = O.compile_ops(ts, fsm, fr.size)
    # host numpy storage (drop-in for the numba backend)
    st = z["packed"].copy()
    p, info = impl.run_ops(st, np.zeros((0, nt, nt)), op, dst, s1, s2, 0, op.size)
    assert (p, info) == (op.size, -1)
    assert relf(st, z["factor"]) < FACTOR_TOL
    # device storage, split into two calls [0, k) + [k, P)
    dev = torch.from_numpy(z["packed"].copy()).cuda()
    k = op.size // 2
    assert impl.run_ops(dev, None, op, dst, s1, s2, 0, k) == (k, -1)
    assert impl.run_ops(dev, None, op, dst, s1, s2, k, op.size) == (op.size, -1)
    assert relf(dev.cpu().numpy(), z["factor"]) < FACTOR_TOL
    # replay residual on device vs the reference value
    diag = fr == fc
    e2 = impl.replay_residual(st, z["packed"], op, dst, s1, s2, diag)
    bw = np.sqrt(e2 / z["anorm2"])
    assert bw <= BACKWARD_TOL
    ref_bw = np.sqrt(float(z["resid2"]) / z["anorm2"])
    assert bw < 50 * max(ref_bw, 1e-17)
    # tree-reduction stream (ZERO / GEADD / scratch slots)
    o2 = z["ops_tree2"]
    R = int(o2[1].max() - fr.size + 1) if o2[1].max() >= fr.size else 0
    st2 = z["packed"].copy()
    sc = np.zeros((max(R, 1), nt, nt))
    assert impl.run_ops(st2, sc, o2[0].astype(np.int8), o2[1], o2[2], o2[3], 0, o2.shape[1]) == (o2.shape[1], -1)
    assert relf(st2, z["factor_tree2"]) < FACTOR_TOL


def test_run_ops_failure_semantics(torch):
    *_, impl = _imports()
    z = load_case("b200")
    n, nt = int(z["n"]), int(z["nt"])
    fr, fc, fsm, _ = O.tile_symbolic(n, nt, z["g_rows"], z["g_cols"])
    op, dst, s1, s2, _ = O.compile_ops(O.task_stream(fsm.shape[0], fsm), fsm, fr.size)
    bad = z["packed"].copy()
    k = 5
    s = fsm[k, k]
    bad[s, 3, 3] = -50.0  # local pivot 3 of tile 5 becomes negative
    ref = bad.copy()
    pr, ir = O.run_ops(ref, np.zeros((0, nt, nt)), op, dst, s1, s2, 0, op.size)
    p, info = impl.run_ops(bad, None, op, dst, s1, s2, 0, op.size)
    assert (p, info) == (pr, ir) and ir >= 0
    with pytest.raises(ValueError):
        impl.run_ops(bad, None, op, dst + 10_000, s1, s2, 0, op.size)


# ------------------------------------------------------- optimised path --
def _pm(z):
    from paper_2501_02483_b200 import matcore
    return matcore.SymmetricCsc(int(z["n"]), z["cp"], z["ri"], z["vals"])


def _check_ctx(api, ctsf, symbolic, impl, ctx, z, m):
    n = m.n
    # factor vs the live reference factor (same ordering, same tile grid)
    got = ctx.factor.host_storage()
    assert got.shape == z["factor"].shape
    assert relf(got, z["factor"]) < FACTOR_TOL
    # backward error through the device replay of the sequential stream
    op, dst, s1, s2, _ = symbolic.compile_ops(ctx.symbolic, 0)
    fg = ctx.symbolic.factor_grid
    from paper_2501_02483_b200 import matcore
    pm = matcore.SymmetricCsc(n, z["pcp"], z["pri"], z["pvals"])
    tpl = ctsf.pack_into_grid(pm, fg).storage
    e2 = impl.replay_residual(ctx.factor.storage, tpl, op, dst, s1, s2, fg.tile_rows == fg.tile_cols)
    assert np.sqrt(e2) / anorm_f(m.col_ptr, m.values) <= BACKWARD_TOL
    ld = api.logdet(ctx)
    assert abs(ld - float(z["logdet_dense"])) <= LOGDET_TOL * max(1.0, abs(float(z["logdet_dense"])))
    x = api.solve(ctx, z["rhs"])
    A = O.dense_of(n, m.col_ptr, m.row_idx, m.values)
    assert np.linalg.norm(A @ x - z["rhs"]) / np.linalg.norm(z["rhs"]) <= SOLVE_TOL
    assert np.allclose(x, z["x"], rtol=0, atol=1e-10 * np.abs(z["x"]).max())


@pytest.mark.parametrize("name", CASE_NAMES)
def test_factorize_plan_path(torch, name):
    api, ctsf, matcore, symbolic, impl = _imports()
    z = load_case(name)
    m = _pm(z)
    ctx = api.factorize(m, api.FactorOptions(tile_size=int(z["nt"])))
    assert np.array_equal(ctx.permutation.forward, z["sel"])
    _check_ctx(api, ctsf, symbolic, impl, ctx, z, m)


@pytest.mark.parametrize("variant", [
    dict(tree_reduction="off"), dict(lookahead=False), dict(lookahead=3), dict(lookahead=3, executor="graph"), dict(executor="direct"), dict(executor="graph"),
    dict(workers=2, tree_reduction="on"), dict(workers=4, chunk=3, tree_reduction="on"),
    dict(workers=16, chunk=1, tree_reduction="on"), dict(workers=2, tree_reduction="on", executor="graph")])
def test_factorize_plan_variants(torch, variant):
    api, ctsf, matcore, symbolic, impl = _imports()
    for name in ("d1000", "f48", "c500bd"):
        z = load_case(name)
        m = _pm(z)
        ctx = api.factorize(m, api.FactorOptions(tile_size=int(z["nt"]), **variant))
        _check_ctx(api, ctsf, symbolic, impl, ctx, z, m)


def test_graph_and_direct_bitwise_and_batch_isolation(torch):
    api, ctsf, matcore, *_ = _imports()
    z = load_case("d1000")
    m = _pm(z)
    nt = int(z["nt"])
    # deterministic: fixed summation orders, no atomics on data.  Graph and
    # direct launch the same kernels; the persistent executor uses 256-thread
    # update variants (different split-K reduction order) -> equal within FP.
    a = api.factorize(m, api.FactorOptions(tile_size=nt)).factor.host_storage()
    a2 = api.factorize(m, api.FactorOptions(tile_size=nt)).factor.host_storage()
    b = api.factorize(m, api.FactorOptions(tile_size=nt, executor="direct")).factor.host_storage()
    c = api.factorize(m, api.FactorOptions(tile_size=nt, executor="graph")).factor.host_storage()
    assert np.array_equal(a, a2) and np.array_equal(b, c)
    assert relf(a, b) < FACTOR_TOL
    ms = []
    for seed in range(5):
        v = m.values * (1.0 + 0.01 * seed)
        ms.append(matcore.SymmetricCsc(m.n, m.col_ptr, m.row_idx, v))
    solo = [api.factorize(x, api.FactorOptions(tile_size=nt)).factor.host_storage() for x in ms]
    many = api.factorize_many(ms, api.FactorOptions(tile_size=nt), lanes=3)
    for s, c in zip(solo, many):
        assert np.array_equal(s, c.factor.host_storage())


def test_not_positive_definite_reports_indices(torch):
    api, ctsf, matcore, *_ = _imports()
    from paper_2501_02483_b200.errors import FactorizeManyError, NotPositiveDefiniteError
    z = load_case("e2000s")  # RCM-permuted case: original index differs
    m = _pm(z)
    vals = m.values.copy()
    j = 1234
    vals[m.col_ptr[j]] = 1e-3  # diagonal no longer dominant -> indefinite
    bad = matcore.SymmetricCsc(m.n, m.col_ptr, m.row_idx, vals)
    nt = int(z["nt"])
    # oracle: first failing pivot of the same permuted stream
    fwd = z["sel"]
    pcp, pri, pv = O.permute(m.n, m.col_ptr, m.row_idx, vals, fwd)
    fr, fc, fsm, _ = O.tile_symbolic(m.n, nt, z["g_rows"], z["g_cols"])
    st = O.pack(m.n, nt, pcp, pri, pv, fsm, fr.size)
    op, dst, s1, s2, _ = O.compile_ops(O.task_stream(fsm.shape[0], fsm), fsm, fr.size)
    p, info = O.run_ops(st, np.zeros((0, nt, nt)), op, dst, s1, s2, 0, op.size)
    assert info >= 0
    assert op[p] == O.POTRF
    want = int(fr[dst[p]]) * nt + info
    with pytest.raises(NotPositiveDefiniteError) as ei:
        api.factorize(bad, api.FactorOptions(tile_size=nt))
    e = ei.value
    assert e.index == want
    inv = np.empty_like(fwd)
    inv[fwd] = np.arange(m.n)
    assert e.original_index == int(inv[want])
    with pytest.raises(FactorizeManyError) as ee:
        api.factorize_many([m, bad, m], api.FactorOptions(tile_size=nt))
    assert set(ee.value.errors) == {1}
    assert ee.value.results[0] is not None and ee.value.results[2] is not None


@pytest.mark.parametrize("nt", [8, 16, 40, 48, 64, 96, 120, 160, 240])
def test_tile_size_sweep_properties(torch, nt):
    """Size-independent properties at n=3000 across tile sizes."""
    api, ctsf, matcore, symbolic, impl = _imports()
    m = matcore.generate_arrowhead(matcore.ArrowheadSpec(3000, 60, 20, seed=3))
    ctx = api.factorize(m, api.FactorOptions(tile_size=nt, ordering="identity"))
    op, dst, s1, s2, _ = symbolic.compile_ops(ctx.symbolic, 0)
    fg = ctx.symbolic.factor_grid
    tpl = ctsf.pack_into_grid(m, fg).storage
    e2 = impl.replay_residual(ctx.factor.storage, tpl, op, dst, s1, s2, fg.tile_rows == fg.tile_cols)
    assert np.sqrt(e2) / anorm_f(m.col_ptr, m.values) <= BACKWARD_TOL
    sign, ld = np.linalg.slogdet(m.to_dense())
    assert abs(api.logdet(ctx) - ld) <= LOGDET_TOL * abs(ld)
    b = np.random.default_rng(nt).standard_normal(m.n)
    x = api.solve(ctx, b)
    A = m.to_dense()
    assert np.linalg.norm(A @ x - b) / np.linalg.norm(b) <= SOLVE_TOL


def test_c1_config_end_to_end(torch):
    """BASELINE config 1 (n=10000, b=200, t=50, nt=120) vs the oracle factor."""
    api, ctsf, matcore, symbolic, impl = _imports()
    m = matcore.generate_arrowhead(matcore.ArrowheadSpec(10_000, 200, 50, seed=0))
    nt = 120
    ctx = api.factorize(m, api.FactorOptions(tile_size=nt))
    assert ctx.permutation.is_identity()
    fg = ctx.symbolic.factor_grid
    fsm = fg.slot_map
    ts = O.task_stream(fsm.shape[0], fsm)
    op, dst, s1, s2, _ = O.compile_ops(ts, fsm, fg.n_tiles)
    tpl = ctsf.pack_into_grid(m, fg).storage
    ref = tpl.copy()
    O.run_ops(ref, np.zeros((0, nt, nt)), op, dst, s1, s2, 0, op.size)
    assert relf(ctx.factor.host_storage(), ref) < FACTOR_TOL
    e2 = impl.replay_residual(ctx.factor.storage, tpl, op, dst, s1, s2, fg.tile_rows == fg.tile_cols)
    assert np.sqrt(e2) / anorm_f(m.col_ptr, m.values) <= BACKWARD_TOL
    ld_ref = O.logdet(ref, fsm, m.n, nt)
    assert abs(api.logdet(ctx) - ld_ref) <= LOGDET_TOL * abs(ld_ref)
    b = np.ones(m.n)
    x = api.solve(ctx, b)
    xr = O.tile_solve(ref, fsm, m.n, nt, b)
    assert np.linalg.norm(x - xr) / np.linalg.norm(xr) <= SOLVE_TOL


def _vs_oracle(m, nt, **opts):
    """Factor through the public API and check factor / backward error /
    logdet / solve against the oracle executor on the same inputs."""
    api, ctsf, matcore, symbolic, impl = _imports()
    ctx = api.factorize(m, api.FactorOptions(tile_size=nt, **opts))
    fg = ctx.symbolic.factor_grid
    fsm = fg.slot_map
    op, dst, s1, s2, _ = O.compile_ops(O.task_stream(fsm.shape[0], fsm), fsm, fg.n_tiles)
    assert ctx.permutation.is_identity()
    pm = m
    tpl = ctsf.pack_into_grid(pm, fg).storage
    ref = tpl.copy()
    p, info = O.run_ops(ref, np.zeros((0, nt, nt)), op, dst, s1, s2, 0, op.size)
    assert info == -1
    assert relf(ctx.factor.host_storage(), ref) < FACTOR_TOL
    e2 = impl.replay_residual(ctx.factor.storage, tpl, op, dst, s1, s2, fg.tile_rows == fg.tile_cols)
    assert np.sqrt(e2) / anorm_f(pm.col_ptr, pm.values) <= BACKWARD_TOL
    ld_ref = O.logdet(ref, fsm, pm.n, nt)
    assert abs(api.logdet(ctx) - ld_ref) <= LOGDET_TOL * abs(ld_ref)


@pytest.mark.parametrize("nt", [40, 64, 120, 160, 240])
@pytest.mark.parametrize("occ", [1, 2])
def test_inla_small_with_fill(torch, nt, occ, monkeypatch):
    """Small INLA precision (block-tridiagonal + arrow, fill tiles) through the
    persistent executor, both occupancies (fused diagonal SYRK streaming)."""
    from paper_2501_02483_b200 import workloads as W
    if occ == 2:
        monkeypatch.setenv("TILECHOL_EXPERIMENTAL", "1")  # gated mode
    m = W.InlaFamily(nx=10, ny=12, nsteps=20, nfix=3).matrix(0.5, 0.9, 1e-3)
    _vs_oracle(m, nt, ordering="identity", occupancy=occ)


@pytest.mark.parametrize("occ", [1, 2])
def test_variable_band_small(torch, occ, monkeypatch):
    if occ == 2:
        monkeypatch.setenv("TILECHOL_EXPERIMENTAL", "1")
    from paper_2501_02483_b200 import workloads as W
    m = W.c2_variable_band(n=6000, t=40, seg_len=600, max_band=300)
    _vs_oracle(m, 48, ordering="identity", occupancy=occ)


def test_inla_batch_device_assembly_and_streaming_logdets(torch):
    """C5 machinery on a small INLA family: device value assembly
    (tc_plan_pack_lincomb) is bitwise the host values; the streaming batch
    (logdet_many, lanes sharing the GPU) reproduces solo log-determinants
    bitwise and aggregates a failing member without cancelling the others."""
    from paper_2501_02483_b200 import workloads as W
    from paper_2501_02483_b200.errors import FactorizeManyError, NotPositiveDefiniteError
    api, ctsf, matcore, symbolic, impl = _imports()
    fam = W.InlaFamily(nx=10, ny=12, nsteps=20, nfix=3)
    thetas = W.c5_thetas()[::11]
    ms = [fam.matrix(*t) for t in thetas]
    opts = api.FactorOptions(tile_size=64)
    solo = np.array([api.logdet(api.factorize(m, opts)) for m in ms])
    many = api.logdet_many(ms, opts, lanes=3)
    assert np.array_equal(solo, many)
    pat = api._pattern_for(ms[0], opts)
    plan = pat.plan
    offs = pat.offsets()
    sh = torch.cuda.current_stream().cuda_stream
    for t, m in zip(thetas, ms):
        coef, basis = fam.lincomb(*t)
        bd = torch.from_numpy(np.stack([pat.permuted_values(matcore.SymmetricCsc(m.n, m.col_ptr, m.row_idx, b))
                                        for b in basis])).cuda()
        s1, s2 = plan.new_storage(), plan.new_storage()
        plan.pack_lincomb(bd, coef, offs, s1, sh)
        plan.pack(torch.from_numpy(np.ascontiguousarray(pat.permuted_values(m))).cuda(), offs, s2, sh)
        assert torch.equal(s1, s2)
    bad = matcore.SymmetricCsc(ms[1].n, ms[1].col_ptr, ms[1].row_idx, -ms[1].values)
    with pytest.raises(FactorizeManyError) as ei:
        api.logdet_many([ms[0], bad, ms[2]], opts, lanes=2)
    assert set(ei.value.errors) == {1} and isinstance(ei.value.errors[1], NotPositiveDefiniteError)
    assert ei.value.results[0] == solo[0] and ei.value.results[2] == solo[2]


# ------------------------------------------------- device solve (persistent) --
@pytest.mark.parametrize("nt,k", [(17, 1), (48, 3), (120, 11), (200, 2), (240, 1), (480, 1)])
def test_solve_persistent_sweep(torch, nt, k):
    """tc_plan_solve: batched L_kk^-T + one persistent launch for both sweeps;
    residual <= 1e-10 against the CSC matrix for k right-hand sides (k > 8
    exercises the right-hand-side chunking), equal to the oracle tile solve."""
    api, ctsf, matcore, symbolic, impl = _imports()
    m = matcore.generate_arrowhead(matcore.ArrowheadSpec(n=3001, b=90, t=13, seed=3))
    ctx = api.factorize(m, api.FactorOptions(tile_size=nt))
    rng = np.random.default_rng(nt)
    b = rng.standard_normal((m.n, k)) if k > 1 else rng.standard_normal(m.n)
    x = api.solve(ctx, b)
    A = O.dense_of(m.n, m.col_ptr, m.row_idx, m.values)
    res = np.linalg.norm(A @ x - b) / np.linalg.norm(b)
    assert res <= SOLVE_TOL, res
    fg = ctx.symbolic.factor_grid
    st = ctx.factor.host_storage()
    xr = O.tile_solve(st, fg.slot_map, m.n, nt, b[:, 0] if k > 1 else b, fwd=ctx.permutation.forward)
    x0 = x[:, 0] if k > 1 else x
    assert np.linalg.norm(x0 - xr) <= 1e-12 * np.linalg.norm(xr)
    # deterministic: the same solve twice is bitwise equal
    assert np.array_equal(api.solve(ctx, b), x)


def test_solve_many_streaming_and_sharded_single_rank(torch):
    """Streaming batch with device solves (api.solve_many, the C5 path) equals
    solo factorize + solve, and logdet_many_sharded(rhs=...) on one rank
    returns the same rows."""
    from paper_2501_02483_b200 import workloads as W
    api, *_ = _imports()
    fam = W.InlaFamily(nx=10, ny=12, nsteps=20, nfix=3)
    ms = [fam.matrix(*t) for t in W.c5_thetas()[::9]]
    opts = api.FactorOptions(tile_size=64)
    b = np.linspace(-1.0, 1.0, ms[0].n)
    solo_ld, solo_x = [], []
    for m in ms:
        c = api.factorize(m, opts)
        solo_ld.append(api.logdet(c))
        solo_x.append(api.solve(c, b))
    ld, X = api.solve_many(ms, b, opts, lanes=3)
    assert np.array_equal(ld, np.array(solo_ld))
    assert np.array_equal(X, np.stack(solo_x))
    ld2, X2 = api.logdet_many_sharded(ms, opts, lanes=2, rhs=b)
    assert np.array_equal(ld2, ld) and np.array_equal(X2, X)
    for m, x in zip(ms, X):
        A = O.dense_of(m.n, m.col_ptr, m.row_idx, m.values)
        assert np.linalg.norm(A @ x - b) <= SOLVE_TOL * np.linalg.norm(b)
