"""The LEO-campaign oracle (oracle/leo.py) pinned to the reference's own
outputs (tests/golden/leo_*.npz, made by tests/golden/gen_golden_leo.py):
beam selection indices, per-step decisions, ranks, costs and rates of the
reference harness's run_campaign / run_trial."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import leo as OL
from paper_2512_16543_b200.leo import ScenarioConfig, complexity_curve, ecdf

from conftest import load_golden


def cfg_from(g) -> ScenarioConfig:
    kw = {}
    for k in g.files:
        if k.startswith("cfg_"):
            v = g[k]
            kw[k[4:]] = tuple(float(x) for x in v) if k == "cfg_eta_list" else v.item()
    return ScenarioConfig(**kw).validate()


def test_beam_selection_matches_reference():
    g = load_golden("leo_beams")
    for i in range(int(g["n_cases"])):
        cols = OL.pick_beams(g[f"power_{i}"], int(g[f"nrf_{i}"]))
        assert np.array_equal(cols, g[f"cols_{i}"]), i


@pytest.mark.parametrize("name", ["leo_small", "leo_rect", "leo_default"])
def test_campaign_matches_reference(name):
    g = load_golden(name)
    cfg = cfg_from(g)
    assert np.isclose(OL.alpha_of(cfg), float(g["alpha"]), rtol=1e-15)
    out = OL.campaign(cfg)
    labels = list(g["labels"])
    assert out["labels"] == labels
    for i, lab in enumerate(labels):
        for b, dec in enumerate(out["decisions"][lab]):
            assert np.array_equal(dec, g[f"decisions_{i}"][b]), (lab, b)
        assert out["mean_cost"][lab] == float(g[f"mean_cost_{i}"])
        assert out["mean_k"][lab] == float(g[f"mean_k_{i}"])
        assert [out["counts"][lab][k] for k in ("full", "woodbury", "none")] == \
            list(g[f"counts_{i}"])
        np.testing.assert_allclose(out["pooled"][lab], g[f"pooled_{i}"], rtol=1e-9, atol=0)
        np.testing.assert_allclose(out["trial_means"][lab], g[f"trial_means_{i}"], rtol=1e-9)
    tab = np.array([[r[2], r[3]] for r in out["table"]])
    np.testing.assert_allclose(tab, g["table"], rtol=1e-6, atol=1e-9)


@pytest.mark.parametrize("name", ["leo_small", "leo_rect", "leo_default"])
def test_snapshots_match_reference(name):
    g = load_golden(name)
    cfg = cfg_from(g)
    snaps = []
    OL.sweep_trial(cfg, [("conventional", None)], 0, cfg.seed, keep_snaps=snaps)
    cols = np.stack([s[2] for s in snaps])
    assert np.array_equal(cols, g["cols"])
    for j, t in enumerate(g["snap_steps"]):
        np.testing.assert_allclose(snaps[t][0], g["H_eff"][j], rtol=0, atol=1e-13)
        scale = np.abs(g["Hr"][j]).max()
        np.testing.assert_allclose(snaps[t][1], g["Hr"][j], rtol=0, atol=1e-12 * scale)


@pytest.mark.parametrize("name", ["leo_small", "leo_rect"])
def test_single_trial_records_match_reference(name):
    g = load_golden(name)
    cfg = cfg_from(g)
    labels = list(g["labels"])
    etas = [None] + sorted(set(cfg.eta_list), reverse=True)
    for i, (lab, eta) in enumerate(zip(labels, etas)):
        run = OL.sweep_trial(cfg, [(lab, eta)], 1, cfg.seed)[lab]
        assert np.array_equal(np.array(run.methods, np.uint8), g[f"trial_method_{i}"])
        assert np.array_equal(np.array(run.k_est), g[f"trial_k_{i}"])
        assert np.array_equal(np.array(run.costs), g[f"trial_cost_{i}"])
        np.testing.assert_allclose(run.rates, g[f"trial_rates_{i}"], rtol=1e-9)


def test_full_default_pass_prefix_matches_reference():
    """The default 120 s pass: beams of every step, and the first 150 steps of
    the conventional and eta=0.9 runs (the oracle is serial numpy)."""
    g = load_golden("leo_full_trial")
    cfg = ScenarioConfig().validate()
    T = 150
    snaps = []
    runs = OL.sweep_trial(cfg, [("conventional", None), ("wb_arsvd_eta0.9", 0.9)], 0, cfg.seed,
                          keep_snaps=snaps, steps=T)
    assert np.array_equal(np.stack([s[2] for s in snaps]), g["cols"][:T])
    for i, lab in enumerate(("conventional", "wb_arsvd_eta0.9")):
        r = runs[lab]
        assert np.array_equal(np.array(r.methods, np.uint8), g[f"trial_method_{i}"][:T])
        assert np.array_equal(np.array(r.k_est), g[f"trial_k_{i}"][:T])
        np.testing.assert_allclose(r.rates, g[f"trial_rates_{i}"][:T], rtol=1e-9)


def test_elevation_mask_raises():
    cfg = ScenarioConfig(K=1, N_RF=1).validate()
    far = np.array([[6371e3 * np.cos(np.radians(40.0)), 6371e3 * np.sin(np.radians(40.0)), 0.0]])
    with pytest.raises(OL.OracleBelowMask):
        OL.orbit(cfg, far, 60.0)


def test_ecdf_and_complexity_curve():
    e = ecdf([3.0, 1.0, 2.0, 2.0])
    assert np.array_equal(e, np.array([[1.0, 0.25], [2.0, 0.75], [3.0, 1.0]]))
    c = complexity_curve(16)
    assert c.shape == (16, 2) and c[0, 0] == 1.0
    assert np.isclose(c[7, 1], (256 + 256 * 8 + 512 + 64 * 16) / 4096)
