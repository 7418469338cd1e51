"""Drop-in proof: the reference's own harness, installed
unmodified in baseline/_ref, runs its per-trial sweep with the numerical core
swapped for this package -- harness.lowrank, harness.rzf_precoder and
harness.sum_rate rebound exactly as INTEGRATION.md shows
(harness.py:22,25,232-243) -- and reproduces its own numpy results: same
dispatcher decisions, ranks and cost units, sum-rates to 1e-9.  The
exceptions it catches are the reference's classes (errors.py:28-50)."""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def leorzf():
    if not (REF / "leorzf").exists():
        pytest.skip("reference not installed in baseline/_ref (pip install --target)")
    sys.path.insert(0, str(REF))
    import leorzf.harness  # noqa: F401
    return sys.modules["leorzf"]


def _cfg(leorzf):
    from leorzf.config import ScenarioConfig
    return ScenarioConfig(K=4, n_x=4, n_y=4, N_RF=6, pass_s=3.0, update_rate_Hz=10.0,
                          mc_runs=2, eta_list=(0.9, 0.65), n_reset=12).validate()


def test_reference_sweep_runs_on_the_b200_core(cuda, leorzf, monkeypatch):
    import leorzf.harness as H
    import paper_2512_16543_b200 as b200
    cfg = _cfg(leorzf)
    specs = [("conventional", None), ("wb_arsvd_eta0.9", 0.9), ("wb_arsvd_eta0.65", 0.65)]
    ref = H._sweep_trial(cfg, specs, 1, cfg.seed, collect_records=True, collect_decisions=True)
    monkeypatch.setattr(H, "lowrank", b200)
    monkeypatch.setattr(H, "rzf_precoder", b200.rzf_precoder)
    monkeypatch.setattr(H, "sum_rate", b200.sum_rate)
    got = H._sweep_trial(cfg, specs, 1, cfg.seed, collect_records=True, collect_decisions=True)
    for lab, _ in specs:
        r, g = ref[lab], got[lab]
        assert g.decisions == r.decisions, lab
        assert [s.k_est for s in g.records] == [s.k_est for s in r.records], lab
        assert g.total_cost == r.total_cost, lab
        np.testing.assert_allclose(g.rates, r.rates, rtol=1e-9)
    assert sum(1 for d in got["wb_arsvd_eta0.65"].decisions if d == 1) > 0   # Woodbury steps ran
