"""Batched trajectory runner on the GPU vs the reference-generated golden
trajectories (C1, C2 samples) and vs the oracle sweep run live; full-size
C2 checked through size-independent properties."""

import numpy as np
import pytest
import torch

from conftest import load_golden, rel
from oracle import port, sweep
from paper_2512_16543_b200 import TrajectoryConfig, run_trajectory, scenario as S
from paper_2512_16543_b200.omega import OmegaStreams

pytestmark = pytest.mark.gpu


def _cfg(spec, eta):
    return TrajectoryConfig(alpha=spec.alpha, eta=eta, k_init=spec.k_init, p=spec.p,
                            i_max=spec.i_max)


def _run(spec, H, eta, trials, chunk=None, keep=True):
    st = None if eta is None else OmegaStreams.for_method(spec.seed, eta, trials)
    return run_trajectory(H, S.noise_vector(spec), _cfg(spec, eta), st, chunk=chunk,
                          keep_A_inv=keep)


def _compare(res, b, g, pre, T, a_tol, rate_tol):
    assert np.array_equal(res.method[b], g[pre + "method"]), pre
    assert np.array_equal(res.k_est[b], g[pre + "k_est"]), (pre, res.k_est[b], g[pre + "k_est"])
    assert np.array_equal(res.consumed[b], g[pre + "consumed"]), pre
    assert np.max(np.abs(res.rates[b] - g[pre + "rates"]) / np.abs(g[pre + "rates"])) < rate_tol
    if pre + "A_inv" in g:
        err = max(rel(res.A_inv[b, t], g[pre + "A_inv"][t]) for t in range(T))
        assert err < a_tol, (pre, err)


@pytest.mark.parametrize("eta", [None, 0.999, 0.9, 0.8, 0.65])
def test_C1_matches_reference(cuda, eta):
    g = load_golden("traj_C1")
    H = g["t0_H"][None]
    res = _run(S.C1, H, eta, [0])
    lab = "full" if eta is None else f"e{int(round(eta * 1000))}"
    _compare(res, 0, g, f"t0_{lab}_", 50, 1e-10, 1e-10)
    if eta is not None:
        assert res.cost[0].sum() > 0


@pytest.mark.parametrize("chunk", [1, 7, 50])
def test_C1_chunking_invariant(cuda, chunk):
    g = load_golden("traj_C1")
    H = g["t0_H"][None]
    res = _run(S.C1, H, 0.9, [0], chunk=chunk)
    _compare(res, 0, g, "t0_e900_", 50, 1e-10, 1e-10)


@pytest.mark.parametrize("tag,spec,eta,a_tol,r_tol", [
    ("C2s", S.C2, None, 1e-10, 1e-10),
    ("C2s", S.C2, 0.999, 1e-10, 1e-10),
    ("C2s", S.C2, 0.9, 1e-10, 1e-10),
    ("C2s_c64", S.C2.with_(dtype="c64"), None, 1e-4, 1e-4),
    ("C2s_c64", S.C2.with_(dtype="c64"), 0.9, 1e-4, 1e-4),
    ("C2s_snr0", S.C2.with_(snr_db=0.0), 0.9, 1e-10, 1e-10),
    ("C2s_snr20", S.C2.with_(snr_db=20.0), 0.9, 1e-10, 1e-10),
])
def test_C2_samples_match_reference(cuda, tag, spec, eta, a_tol, r_tol):
    g = load_golden("traj_" + tag)
    trials = [0, 1] if tag == "C2s" else [0]
    H = S.channels(spec, trials=trials, t1=24)
    res = _run(spec, H, eta, trials)
    lab = "full" if eta is None else f"e{int(round(eta * 1000))}"
    for b in trials:
        _compare(res, b, g, f"t{b}_{lab}_", 24, a_tol, r_tol)


def test_C2_full_size_properties_and_oracle_spot_check(cuda):
    """B=64, T=200 (the bench workload): every step finite, WB = full at
    eta=0.999, and two trials replayed step-for-step by the oracle."""
    spec = S.C2
    H = S.channels(spec)
    res = _run(spec, H, spec.eta, list(range(spec.B)), keep=False)
    full = _run(spec, H, None, list(range(spec.B)), keep=False)
    assert np.all(np.isfinite(res.rates)) and np.all(res.rates > 0)
    # the capped schedule never reaches 99.9 % energy -> fallback r = 21 > K/2 -> full
    assert np.all(res.method[:, 1:] == 0) and np.all(res.k_est[:, 1:] == 21)
    assert np.allclose(res.rates, full.rates, rtol=1e-12)
    for b in (0, 37):
        sk = np.random.default_rng(S.stream_seed(spec.seed, S.method_label(spec.eta), b))
        ref = sweep.sweep_trial(H[b], spec.alpha, S.noise_vector(spec), 1.0,
                                port.Cfg(spec.eta, spec.k_init, spec.p, spec.i_max), sk)
        assert np.array_equal(res.k_est[b], ref.k_est)
        assert np.array_equal(res.consumed[b], ref.consumed)
        assert np.allclose(res.rates[b], ref.rates, rtol=1e-10)


def test_C2_eta09_woodbury_chain_vs_oracle(cuda):
    spec = S.C2.with_(B=4, T=60)
    H = S.channels(spec)
    res = _run(spec, H, 0.9, list(range(4)), chunk=25)
    assert np.mean(res.method[:, 1:] == 1) > 0.9
    for b in range(4):
        sk = np.random.default_rng(S.stream_seed(spec.seed, S.method_label(0.9), b))
        ref = sweep.sweep_trial(H[b], spec.alpha, S.noise_vector(spec), 1.0,
                                port.Cfg(0.9, spec.k_init, spec.p, spec.i_max), sk,
                                keep_state=True)
        tie = ref.margin < 1e-9
        ok = (res.k_est[b] == ref.k_est) | tie
        assert ok.all(), (b, np.nonzero(~ok))
        if (res.k_est[b] == ref.k_est).all():
            err = max(rel(res.A_inv[b, t], ref.A_inv[t]) for t in range(spec.T))
            assert err < 1e-10, err
            assert np.allclose(res.rates[b], ref.rates, rtol=1e-10)


@pytest.mark.parametrize("delta,via_gram", [("formula", False), ("diff", True), ("formula", True)])
def test_C2_runner_variants_match_reference(cuda, delta, via_gram):
    """Gram-correction form (formula vs differenced Grams) and rate form
    (H W vs (G - alpha I) A^-1) all reproduce the reference trajectory."""
    g = load_golden("traj_C2s")
    spec = S.C2
    H = S.channels(spec, trials=[0, 1], t1=24)
    cfg = _cfg(spec, 0.9)
    cfg.delta, cfg.rate_via_gram = delta, via_gram
    res = run_trajectory(H, S.noise_vector(spec), cfg, OmegaStreams.for_method(0, 0.9, [0, 1]),
                         keep_A_inv=True)
    for b in (0, 1):
        _compare(res, b, g, f"t{b}_e900_", 24, 1e-10, 1e-10)


@pytest.mark.parametrize("name,B,T,dtype,etas", [
    ("C3", 2, 10, "c64", (0.999, 0.9)),
    ("C4", 2, 6, "c64", (0.999, 0.9)),
    ("C5", 1, 4, "c64", (0.999, 0.9)),
    ("C5", 1, 3, "c128", (0.999,)),
])
def test_larger_configs_vs_oracle(cuda, name, B, T, dtype, etas):
    """C3-C5 shapes (K = 64 / 128 / 256, N = 1024 / 4096) at reduced B and T,
    every method replayed by the oracle on the identical inputs."""
    spec = S.CONFIGS[name].with_(B=B, T=T, dtype=dtype)
    H = S.channels(spec)
    tol = 1e-10 if dtype == "c128" else 1e-4
    for eta in (None,) + etas:
        res = _run(spec, H, eta, list(range(B)))
        for b in range(B):
            cfg = None if eta is None else port.Cfg(eta, spec.k_init, spec.p, spec.i_max)
            sk = None if eta is None else np.random.default_rng(
                S.stream_seed(spec.seed, S.method_label(eta), b))
            ref = sweep.sweep_trial(H[b], spec.alpha, S.noise_vector(spec), 1.0, cfg, sk,
                                    keep_state=True)
            tie = ref.margin < 1e-6 if dtype == "c64" else ref.margin < 1e-9
            assert ((res.k_est[b] == ref.k_est) | tie).all(), (name, eta, res.k_est[b], ref.k_est)
            if not (res.k_est[b] == ref.k_est).all():
                continue
            assert np.array_equal(res.method[b], ref.method), (name, eta)
            assert np.array_equal(res.consumed[b], ref.consumed), (name, eta)
            err = max(rel(res.A_inv[b, t], ref.A_inv[t]) for t in range(T))
            assert err < tol, (name, eta, err)
            assert np.max(np.abs(res.rates[b] / ref.rates - 1)) < tol, (name, eta)


def test_per_user_noise_vector_reaches_every_trial(cuda):
    """sigma_k^2 differs per user (precoding.py:55-80 takes a noise vector): the
    batched runner must apply the same [K] vector to every trial (regression:
    a broadcast [B, K] host array used to reach the kernels Fortran-ordered)."""
    spec = S.C2.with_(B=3, T=10)
    H = S.channels(spec)
    noise = np.linspace(0.05, 0.3, spec.K)
    cfg = _cfg(spec, 0.9)
    res = run_trajectory(H, noise, cfg, OmegaStreams.for_method(spec.seed, 0.9, [0, 1, 2]))
    for b in range(3):
        sk = np.random.default_rng(S.stream_seed(spec.seed, S.method_label(0.9), b))
        ref = sweep.sweep_trial(H[b], spec.alpha, noise, 1.0,
                                port.Cfg(0.9, spec.k_init, spec.p, spec.i_max), sk)
        assert np.array_equal(res.k_est[b], ref.k_est)
        np.testing.assert_allclose(res.rates[b], ref.rates, rtol=1e-10)
