"""Golden fixtures for the hybrid LEO campaign path, produced by the REFERENCE
itself (imported read-only from /root/reference/pkg/src; nothing copied).

    python tests/golden/gen_golden_leo.py

Writes tests/golden/leo_*.npz:

* ``leo_small.npz``   -- a 4-UT / 4x4-array / N_RF=6 scenario with NLOS
  blocks, held beams and periodic resets: the reference's ``run_campaign``
  (pooled rates, per-trial decisions, costs, mean k, counts, table) and
  per-step beam indices / effective channels of trial 0;
* ``leo_rect.npz``    -- a non-square 8x4 array, K = N_RF = 5;
* ``leo_default.npz`` -- the reference's default scenario (K = N_RF = 16,
  16x16 array) over a 6 s pass, 2 trials, all four methods;
* ``leo_full_trial.npz`` -- one full default pass (120 s, 2400 snapshots,
  a reset at 1200) with the conventional method and eta = 0.9;
* ``leo_beams.npz``   -- ``select_beams`` on power tables with ties,
  collisions and fill columns.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

from leorzf import channel as ch  # noqa: E402  (reference, read-only)
from leorzf import harness as hz  # noqa: E402
from leorzf.config import ScenarioConfig  # noqa: E402

SMALL = dict(K=4, n_x=4, n_y=4, N_RF=6, pass_s=2.0, update_rate_Hz=10.0, mc_runs=3,
             eta_list=(0.9, 0.65), n_reset=8, nlos_block_len=3, beam_hold=2)
RECT = dict(K=5, n_x=8, n_y=4, N_RF=5, pass_s=1.5, update_rate_Hz=20.0, mc_runs=2,
            eta_list=(0.8,))
DEFAULT_SHORT = dict(pass_s=6.0, mc_runs=2)


def col_index(F, C):
    """Codebook index of every column of F (exact column match)."""
    out = []
    for c in range(F.shape[1]):
        hit = np.nonzero(np.all(C == F[:, [c]], axis=0))[0]
        assert hit.size == 1
        out.append(int(hit[0]))
    return np.array(out, dtype=np.int64)


def channel_trace(cfg, trial, seed, steps):
    """Replay the harness's channel loop (harness.py:197-226) for one trial and
    record beam indices every step and H_eff / H F_RF at ``steps``."""
    rng = np.random.default_rng(hz.stream_seed(seed, hz.CHANNEL_STREAM, trial))
    ctx = ch.make_pass(cfg, rng)
    dt = 1.0 / cfg.update_rate_Hz
    beams = nlos = None
    cols, heff, hr = [], {}, {}
    for i in range(cfg.n_snapshots):
        if i % cfg.nlos_block_len == 0:
            nlos = ch.draw_nlos(ctx, rng)
        held = beams if (i % cfg.beam_hold != 0) else None
        sn = ch.snapshot(ctx, i * dt, rng, beams=held, nlos_draw=nlos)
        beams = sn.F_RF
        cols.append(col_index(sn.F_RF, ctx.codebook))
        if i in steps:
            heff[i] = sn.H_eff
            hr[i] = sn.H @ sn.F_RF
    return np.stack(cols), np.stack([heff[i] for i in steps]), np.stack([hr[i] for i in steps])


def campaign_arrays(cfg, tag):
    res = hz.run_campaign(cfg, collect_decisions=True)
    out = {"labels": np.array(res.labels)}
    for i, lab in enumerate(res.labels):
        out[f"pooled_{i}"] = res.pooled_rates[lab]
        out[f"trial_means_{i}"] = res.trial_mean_rates[lab]
        out[f"mean_cost_{i}"] = np.array(res.mean_cost[lab])
        out[f"mean_k_{i}"] = np.array(res.mean_k_est[lab])
        out[f"counts_{i}"] = np.array([res.method_counts[lab][k] for k in ("full", "woodbury", "none")])
        out[f"decisions_{i}"] = np.stack(res.decisions[lab])
    out["table"] = np.array([[r.savings_pct, r.degradation_pct] for r in res.table.rows])
    print(tag, {lab: res.method_counts[lab] for lab in res.labels})
    return out


def scenario_arrays(kw):
    cfg = ScenarioConfig(**kw).validate()
    d = {f"cfg_{k}": np.array(v) for k, v in kw.items()}
    d["alpha"] = np.array(cfg.resolved_alpha)
    d["noise"] = np.array(cfg.noise_variance_W)
    return cfg, d


def per_method_trial(cfg, trial, seed, labels_etas):
    out = {}
    for i, (lab, eta) in enumerate(labels_etas):
        r = hz.run_trial(cfg, eta, trial, seed)
        recs = r.snapshots
        out[f"trial_rates_{i}"] = np.array([s.sum_rate for s in recs])
        out[f"trial_method_{i}"] = np.array([hz._DECISION_CODES[s.method] for s in recs], np.uint8)
        out[f"trial_k_{i}"] = np.array([s.k_est for s in recs])
        out[f"trial_cost_{i}"] = np.array([s.cost_units for s in recs])
    return out


def gen_small(name, kw, steps):
    cfg, d = scenario_arrays(kw)
    d.update(campaign_arrays(cfg, name))
    cols, heff, hr = channel_trace(cfg, 0, cfg.seed, steps)
    d.update(cols=cols, snap_steps=np.array(steps), H_eff=heff, Hr=hr)
    etas = sorted(set(cfg.eta_list), reverse=True)
    specs = [(hz.method_label(None), None)] + [(hz.method_label(e), e) for e in etas]
    d.update(per_method_trial(cfg, 1, cfg.seed, specs))
    np.savez_compressed(HERE / f"{name}.npz", **d)


def gen_full_trial():
    cfg, d = scenario_arrays({})
    d.update(per_method_trial(cfg, 0, cfg.seed, [("conventional", None), ("wb_arsvd_eta0.9", 0.9)]))
    cols, heff, hr = channel_trace(cfg, 0, cfg.seed, [0, 1, 1199, 1200, 2399])
    d.update(cols=cols, snap_steps=np.array([0, 1, 1199, 1200, 2399]), H_eff=heff, Hr=hr)
    np.savez_compressed(HERE / "leo_full_trial.npz", **d)


def gen_beams():
    rng = np.random.default_rng(2024)
    geom = ch.ArrayGeometry.uniform_planar(4, 4, 1.0)
    C = ch.dft_codebook(geom)
    cases, out = [], {}
    # random tables, ties (quantised powers), identical UTs, fill columns
    cases.append((rng.random((4, 16)), 4))
    cases.append((np.round(rng.random((5, 16)) * 3) / 3, 8))
    row = rng.random(16)
    cases.append((np.stack([row, row, row]), 3))
    cases.append((np.tile(np.arange(16.0)[::-1] % 4, (6, 1)), 10))
    cases.append((np.zeros((2, 16)), 5))
    for i, (pw, nrf) in enumerate(cases):
        F = ch.select_beams(np.zeros((pw.shape[0], 16)), C, nrf, powers=pw)
        out[f"power_{i}"] = pw
        out[f"nrf_{i}"] = np.array(nrf)
        out[f"cols_{i}"] = col_index(F, C)
    out["n_cases"] = np.array(len(cases))
    np.savez_compressed(HERE / "leo_beams.npz", **out)


def main():
    gen_beams()
    gen_small("leo_small", SMALL, [0, 1, 2, 5, 13, 19])
    gen_small("leo_rect", RECT, [0, 7, 29])
    gen_small("leo_default", DEFAULT_SHORT, [0, 1, 60, 119])
    gen_full_trial()


if __name__ == "__main__":
    main()
