"""The persistent executor's ticket order on a wide-column band plan (the C4
shape: >= 16 tiles per column, chain-first order with the Bd / Md / L_crit /
TRSMc launches of the column chain) must be a
topological order of the launch DAG -- the plan builder otherwise falls back
to creation order silently (TC_DEBUG_ORDER=1 reports it) -- and the factor
must match the graph executor's (same arithmetic, other launch structure)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_wide_band_ticket_order_topological_and_factor(capfd, monkeypatch):
    import torch
    assert torch.cuda.is_available()
    from paper_2501_02483_b200 import api, matcore
    monkeypatch.setenv("TC_DEBUG_ORDER", "1")
    m = matcore.generate_arrowhead(matcore.ArrowheadSpec(12_000, 2400, 60, seed=3))
    o = api.FactorOptions(tile_size=128, ordering="identity")
    api.clear_plan_cache()
    a = api.factorize(m, o).factor.host_storage()
    a2 = api.factorize(m, o).factor.host_storage()
    err = capfd.readouterr().err
    assert "not topological" not in err, err
    assert np.array_equal(a, a2)
    g = api.factorize(m, api.FactorOptions(tile_size=128, ordering="identity", executor="graph")).factor.host_storage()
    assert np.linalg.norm(a - g) / np.linalg.norm(g) < 1e-12
