"""Hybrid LEO campaign on the device (lrz_leo_snapshot, lrz_hybrid_precode_rate,
lrz_campaign_reduce) against the oracle and the reference's own outputs."""

import numpy as np
import pytest
import torch

from oracle import leo as OL
from oracle import port
from paper_2512_16543_b200 import leo as L
from paper_2512_16543_b200 import ops
from paper_2512_16543_b200.errors import BelowMinElevationError

from conftest import load_golden
from test_oracle_leo import cfg_from

pytestmark = pytest.mark.gpu

RTOL_RATE = 1e-9     # per-step sum-rate, relative (complex128 end to end)


@pytest.mark.parametrize("name", ["leo_small", "leo_rect", "leo_default"])
def test_snapshots_match_oracle(cuda, name):
    g = load_golden(name)
    cfg = cfg_from(g)
    trials = [0, 1]
    T = cfg.n_snapshots
    ps = L.DevicePass(cfg, trials, cfg.seed, cuda)
    outs = [ps.generate(t0, min(T, t0 + 7), want_channels=True) for t0 in range(0, T, 7)]
    cat = {k: torch.cat([o[k] for o in outs], 1).cpu().numpy() for k in outs[0]}
    assert not np.any(cat["info"])
    for b, tr in enumerate(trials):
        snaps = []
        OL.sweep_trial(cfg, [("conventional", None)], tr, cfg.seed, keep_snaps=snaps)
        cols = np.stack([s[2] for s in snaps])
        assert np.array_equal(cat["cols"][b], cols)
        if tr == 0:
            assert np.array_equal(cat["cols"][b], g["cols"])
        heff = np.stack([s[0] for s in snaps])
        hr = np.stack([s[1] for s in snaps])
        np.testing.assert_allclose(cat["H_eff"][b], heff, rtol=0, atol=1e-12)
        np.testing.assert_allclose(cat["H_rf"][b], hr, rtol=0, atol=1e-11 * np.abs(hr).max())
    # the channel itself (oracle snapshot at a few steps of trial 0)
    crng = np.random.default_rng(OL.seed_seq(cfg.seed, "channel", 0))
    ps0 = OL.make_pass(cfg, crng)
    nl = None
    for i in range(T):
        if i % cfg.nlos_block_len == 0:
            nl = OL.nlos_draw(cfg, crng)
        if i in (0, T // 2, T - 1):
            sn = OL.snapshot(ps0, i / cfg.update_rate_Hz, nl, cat["cols"][0][i])
            np.testing.assert_allclose(cat["H_tilde"][0, i], sn.H_tilde, rtol=0, atol=1e-12)
            np.testing.assert_allclose(cat["H"][0, i], sn.H, rtol=0,
                                       atol=1e-11 * np.abs(sn.H).max())


@pytest.mark.parametrize("name,chunk", [("leo_small", None), ("leo_small", 3),
                                        ("leo_rect", 11), ("leo_default", 50)])
def test_campaign_matches_reference(cuda, name, chunk):
    g = load_golden(name)
    cfg = cfg_from(g)
    res = L.run_campaign(cfg, collect_decisions=True, chunk=chunk)
    labels = list(g["labels"])
    assert res.labels == labels
    for i, lab in enumerate(labels):
        dec = np.stack(res.decisions[lab])
        assert np.array_equal(dec, g[f"decisions_{i}"]), lab
        assert res.mean_cost[lab] == float(g[f"mean_cost_{i}"])
        assert res.mean_k_est[lab] == float(g[f"mean_k_{i}"])
        assert [res.method_counts[lab][k] for k in ("full", "woodbury", "none")] == \
            list(g[f"counts_{i}"])
        np.testing.assert_allclose(res.pooled_rates[lab], g[f"pooled_{i}"], rtol=RTOL_RATE)
        np.testing.assert_allclose(res.trial_mean_rates[lab], g[f"trial_means_{i}"],
                                   rtol=RTOL_RATE)
    tab = np.array([[r.savings_pct, r.degradation_pct] for r in res.table.rows])
    np.testing.assert_allclose(tab[:, 0], g["table"][:, 0], rtol=0, atol=1e-12)
    np.testing.assert_allclose(tab[:, 1], g["table"][:, 1], rtol=1e-5, atol=1e-8)


def test_run_trial_matches_reference(cuda):
    g = load_golden("leo_small")
    cfg = cfg_from(g)
    etas = [None] + sorted(set(cfg.eta_list), reverse=True)
    for i, eta in enumerate(etas):
        tr = L.run_trial(cfg, eta, 1)
        assert np.array_equal([L.DECISION_CODES[s.method] for s in tr.snapshots],
                              g[f"trial_method_{i}"])
        assert [s.k_est for s in tr.snapshots] == list(g[f"trial_k_{i}"])
        assert [s.cost_units for s in tr.snapshots] == list(g[f"trial_cost_{i}"])
        np.testing.assert_allclose([s.sum_rate for s in tr.snapshots], g[f"trial_rates_{i}"],
                                   rtol=RTOL_RATE)
        assert tr.total_cost_units == float(np.sum(g[f"trial_cost_{i}"]))


def test_full_default_pass_matches_reference(cuda):
    """The reference's default scenario, one whole 120 s pass (2400 snapshots,
    reset at 1200), conventional and eta = 0.9."""
    g = load_golden("leo_full_trial")
    cfg = L.ScenarioConfig().validate()
    specs = [("conventional", None), ("wb_arsvd_eta0.9", 0.9)]
    out = L._simulate(cfg, specs, [0], cfg.seed, cuda, 400, keep_cols=True)
    assert np.array_equal(out["_cols"][0], g["cols"])
    for i, (lab, _) in enumerate(specs):
        r = {k: v.cpu().numpy() for k, v in out[lab].items()}
        assert np.array_equal(r["method"][0], g[f"trial_method_{i}"]), lab
        assert np.array_equal(r["k_est"][0], g[f"trial_k_{i}"]), lab
        np.testing.assert_allclose(r["rates"][0], g[f"trial_rates_{i}"], rtol=RTOL_RATE)
        assert r["stats"][0, 0] == float(np.sum(g[f"trial_cost_{i}"]))


def test_hybrid_precoder_rate_matches_oracle(cuda):
    rng = np.random.default_rng(3)
    K, R, nx, ny = 6, 9, 4, 8
    n_items = 5
    C = OL.codebook(nx, ny)
    H_eff = rng.standard_normal((n_items, K, R)) + 1j * rng.standard_normal((n_items, K, R))
    H = rng.standard_normal((n_items, K, nx * ny)) + 1j * rng.standard_normal((n_items, K, nx * ny))
    cols = np.stack([rng.choice(nx * ny, R, replace=False) for _ in range(n_items)])
    A_inv = np.stack([np.linalg.inv(h @ h.conj().T + 0.3 * np.eye(K)) for h in H_eff])
    noise = rng.uniform(0.1, 1.0, K)
    F_RF = [C[:, c] for c in cols]
    Hr = np.stack([H[i] @ F_RF[i] for i in range(n_items)])
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(cuda)
    out = ops.hybrid_precode_rate(d(H_eff), d(A_inv), d(Hr), d(cols.astype(np.int32)), nx, ny,
                                  d(L.dft_factors(nx, ny)), 2.5,
                                  d(noise.reshape(1, K)), n_items, want_F=True)
    for i in range(n_items):
        F_BB, scale = port.rzf_precoder(H_eff[i], A_inv[i], F_RF[i], 2.5)
        rates, total, _ = port.sum_rate(H[i], F_RF[i], F_BB, noise)
        np.testing.assert_allclose(out["F_BB"][i].cpu().numpy(), F_BB, rtol=1e-12, atol=1e-14)
        assert abs(out["scale"][i].item() - scale) <= 1e-12 * scale
        np.testing.assert_allclose(out["rates"][i].cpu().numpy(), rates, rtol=1e-11)
        assert abs(out["sum"][i].item() - total) <= 1e-11 * total
    assert not out["info"].any()


def test_below_mask_raises(cuda):
    cfg = L.ScenarioConfig(K=4, N_RF=4, n_x=4, n_y=4, pass_s=2.0, footprint_radius_m=3000e3,
                           mc_runs=2).validate()
    with pytest.raises(BelowMinElevationError):
        L.run_campaign(cfg)


def test_campaign_reduce_matches_step_costs(cuda):
    from paper_2512_16543_b200.trajectory import step_costs
    rng = np.random.default_rng(5)
    B, T, K, n_reset = 7, 53, 16, 20
    method = rng.integers(0, 3, (B, T)).astype(np.uint8)
    k = rng.integers(0, K, (B, T)).astype(np.int32)
    tg = np.arange(T)
    reset = (tg == 0) | (tg % n_reset == 0)
    method[:, reset] = 0
    k[:, reset] = 0
    stats = torch.zeros(B, 6, dtype=torch.float64, device=cuda)
    for t0 in (0, 20, 40):
        t1 = min(T, t0 + 20)
        ops.campaign_reduce(torch.from_numpy(method[:, t0:t1].copy()).to(cuda),
                            torch.from_numpy(k[:, t0:t1].copy()).to(cuda), t0, K, n_reset, False,
                            stats)
    st = stats.cpu().numpy()
    cost = step_costs(method, k, np.broadcast_to(~reset, (B, T)), K)
    np.testing.assert_array_equal(st[:, 0], cost.sum(1))
    np.testing.assert_array_equal(st[:, 1], np.where(reset, 0, k).sum(1))
    np.testing.assert_array_equal(st[:, 2], np.full(B, (~reset).sum()))
    for j in range(3):
        np.testing.assert_array_equal(st[:, 3 + j], (method == j).sum(1))


def test_campaign_summary_and_ecdf_on_device(cuda):
    """f4: the pooled means, per-trial means, counts, mean rank / cost and the
    comparison table come from lrz_campaign_summary on the device; the ECDF of
    a CUDA tensor is built on the device (harness.py:95-104, 336-367) -- both
    equal the host computations on the same per-step results."""
    import torch
    from paper_2512_16543_b200 import ops
    cfg = L.ScenarioConfig(K=4, n_x=4, n_y=4, N_RF=6, pass_s=3.0, update_rate_Hz=10.0,
                           mc_runs=3, eta_list=(0.9, 0.65), n_reset=12).validate()
    res = L.run_campaign(cfg, collect_decisions=True, device=cuda)
    for lab in res.labels:
        r = res.per_step[lab]
        np.testing.assert_allclose(res.mean_rate[lab], r["rates"].mean(), rtol=1e-12)
        np.testing.assert_allclose(res.trial_mean_rates[lab], r["rates"].mean(axis=1),
                                   rtol=1e-12)
        st = r["stats"]
        assert res.mean_cost[lab] == pytest.approx(st[:, 0].mean(), rel=1e-14)
        kc = st[:, 2].sum()
        assert res.mean_k_est[lab] == pytest.approx(st[:, 1].sum() / kc if kc else 0.0,
                                                    rel=1e-14)
        assert sum(res.method_counts[lab].values()) == r["rates"].size
        e_dev = L.ecdf(torch.from_numpy(res.pooled_rates[lab]).to(cuda)).cpu().numpy()
        e_host = L.ecdf(res.pooled_rates[lab])
        assert np.array_equal(e_dev, e_host)
    conv = res.labels[0]
    for row in res.table.rows[1:]:
        lab = row.method_label
        assert row.savings_pct == pytest.approx(
            100.0 * (1.0 - res.mean_cost[lab] / res.mean_cost[conv]), rel=1e-12)
        assert row.degradation_pct == pytest.approx(
            100.0 * (1.0 - res.mean_rate[lab] / res.mean_rate[conv]), rel=1e-9, abs=1e-12)
