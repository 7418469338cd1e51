"""The fused C entry points a non-Python caller binds (include/leorzf_b200.h,
SURVEY 8(b)): lrz_update_inverse (the Alg. 2 dispatcher, lowrank.py:319-373)
against the oracle, and lrz_trajectory (one chunk of harness._sweep_trial,
harness.py:221-255, in-order arSVD) against the oracle sweep and the
speculative Python runner, across chunk boundaries."""

import numpy as np
import pytest
import torch

from conftest import rel
from oracle import port, sweep
from paper_2512_16543_b200 import TrajectoryConfig, ops, run_trajectory, scenario as S
from paper_2512_16543_b200.omega import OmegaStreams

pytestmark = pytest.mark.gpu


def test_update_inverse_fused_matches_oracle(cuda):
    spec = S.C2
    H = S.channels(spec, trials=[0, 1], t1=6)
    items = [(H[0, 3], H[0, 4], 0.9), (H[1, 1], H[1, 2], 0.9), (H[0, 4], H[0, 5], 0.999),
             (H[1, 2], H[1, 2], 0.9)]                    # dH = 0: the 'none' branch
    B, K, N = len(items), spec.K, spec.N
    L = 2 * K * 64
    rng = np.random.default_rng(7)
    om = rng.standard_normal((B, L))
    for eta in (0.9, 0.999):
        sel = [i for i, it in enumerate(items) if it[2] == eta]
        Hp = np.stack([items[i][0] for i in sel])
        Hc = np.stack([items[i][1] for i in sel])
        st = [port.gram_matrix(h, spec.alpha) for h in Hp]
        d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(cuda)  # noqa: E731
        out = ops.update_inverse_fused(d(Hp), d(Hc - Hp), spec.alpha,
                                       d(np.stack([s.A for s in st])),
                                       d(np.stack([s.A_inv for s in st])), d(om[sel]),
                                       torch.zeros(len(sel), dtype=torch.int64, device=cuda),
                                       eta, spec.k_init, spec.p, spec.i_max)
        for j, i in enumerate(sel):
            src = port.FlatNormals(om[i])
            ref, method, k, cost, f = port.update_inverse(st[j], Hp[j], Hc[j] - Hp[j],
                                                          port.Cfg(eta, spec.k_init, spec.p,
                                                                   spec.i_max), src)
            code = {"full": 0, "woodbury": 1, "none": 2}[method]
            assert int(out["method"][j]) == code, (i, method)
            assert int(out["k_est"][j]) == k
            assert int(out["consumed"][j]) == src.cursor
            assert float(out["cost"][j]) == cost
            assert rel(out["A_inv"][j].cpu().numpy(), ref.A_inv) < 1e-10
            assert rel(out["A"][j].cpu().numpy(), ref.A) < 1e-12


@pytest.mark.parametrize("name,dtype,eta,B,T,chunks", [
    ("C2", "c128", 0.9, 3, 30, (30,)),
    ("C2", "c128", 0.9, 2, 24, (10, 14)),
    ("C2", "c64", 0.999, 2, 12, (12,)),
    ("C2", "c128", None, 2, 8, (4, 4)),
    ("C3", "c64", 0.9, 2, 10, (5, 5)),
])
def test_trajectory_chunks_match_oracle(cuda, name, dtype, eta, B, T, chunks):
    spec = S.CONFIGS[name].with_(dtype=dtype, B=B, T=T)
    trials = list(range(B))
    H = S.channels(spec)
    K = spec.K
    noise = torch.full((B, K), spec.noise_var, dtype=torch.float64, device=cuda)
    Ai = torch.zeros(B, K, K, dtype=torch.complex128, device=cuda)
    A = torch.zeros_like(Ai)
    streams = None if eta is None else OmegaStreams.for_method(spec.seed, eta, trials)
    G_prev, t0 = None, 0
    got = {k: [] for k in ("rates", "method", "k_est", "consumed", "A_inv")}
    for ch in chunks:
        Hc = torch.from_numpy(np.ascontiguousarray(H[:, t0:t0 + ch])).to(cuda)
        om = None
        if eta is not None:
            L = ch * 2 * K * 64
            om = torch.from_numpy(streams.window(L)).to(cuda)
        out = ops.trajectory_chunk(Hc, spec.alpha, 1.0, noise, t0, 1200, eta, spec.k_init,
                                   spec.p, spec.i_max, om, Ai, A, G_prev, keep_A_inv=True)
        if eta is not None:
            streams.advance(out["consumed"].cpu().numpy())
        G_prev = out["G_last"]
        for k in got:
            got[k].append(out[k].cpu().numpy())
        t0 += ch
    res = {k: np.concatenate(v, axis=1) if k != "consumed" else v for k, v in got.items()}
    tol = 1e-10 if dtype == "c128" else 1e-4
    for b in trials:
        cfg = None if eta is None else port.Cfg(eta, spec.k_init, spec.p, spec.i_max)
        sk = None if eta is None else np.random.default_rng(
            S.stream_seed(spec.seed, S.method_label(eta), b))
        ref = sweep.sweep_trial(H[b], spec.alpha, S.noise_vector(spec), 1.0, cfg, sk,
                                keep_state=True)
        assert np.array_equal(res["k_est"][b], ref.k_est), (b, res["k_est"][b], ref.k_est)
        assert np.array_equal(res["method"][b], ref.method), b
        np.testing.assert_allclose(res["rates"][b], ref.rates, rtol=tol)
        err = max(rel(res["A_inv"][b, t], ref.A_inv[t]) for t in range(T))
        assert err < tol, err
        if eta is not None:
            assert sum(int(c[b]) for c in res["consumed"]) == int(ref.consumed.sum())
    # same per-step results as the speculative Python runner
    cfg = TrajectoryConfig(alpha=spec.alpha, eta=eta, k_init=spec.k_init, p=spec.p,
                           i_max=spec.i_max)
    st2 = None if eta is None else OmegaStreams.for_method(spec.seed, eta, trials)
    py = run_trajectory(H, S.noise_vector(spec), cfg, st2, chunk=chunks[0])
    assert np.array_equal(py.method, res["method"]) and np.array_equal(py.k_est, res["k_est"])
    np.testing.assert_allclose(py.rates, res["rates"], rtol=tol)
