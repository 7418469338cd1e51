"""Runner execution modes against the eager, verified path: CUDA-graph capture
(run_chunk(sync=False)), the in-order arSVD fallback (lrz_arsvd_seq), several
WB methods batched with a per-row eta, and lrz_rng_locate."""

import numpy as np
import pytest
import torch

from conftest import load_golden
from paper_2512_16543_b200 import TrajectoryConfig, TrajectoryRunner, scenario as S
from paper_2512_16543_b200.omega import DeviceOmegaStreams, OmegaStreams

pytestmark = pytest.mark.gpu


def _setup(cuda, spec, eta, trials):
    H = torch.from_numpy(S.channels(spec, trials=trials)).to(cuda)
    noise = torch.full((len(trials), spec.K), spec.noise_var, dtype=torch.float64, device=cuda)
    cfg = TrajectoryConfig(alpha=spec.alpha, eta=eta, k_init=spec.k_init, p=spec.p,
                           i_max=spec.i_max)
    return H, noise, cfg


def test_graph_replay_equals_eager(cuda):
    spec = S.C2.with_(B=8, T=40)
    trials = list(range(8))
    H, noise, cfg = _setup(cuda, spec, spec.eta, trials)
    st = DeviceOmegaStreams.for_method(spec.seed, spec.eta, trials, cuda)
    side = torch.cuda.Stream(cuda)

    def step(sync):
        rn = TrajectoryRunner(8, spec.K, spec.N, torch.complex128, cfg, cuda)
        st.raw.zero_()
        L = spec.T * rn.normals_per_step_max()
        om = st.window(L, stream=side)
        return rn.run_chunk(H, noise, om, omega_ready=st.ready, sync=sync)

    ref = step(True)
    for _ in range(2):
        step(False)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        out = step(False)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert int(out.flags.abs().sum()) == 0
    assert torch.equal(out.method, ref.method)
    assert torch.equal(out.k_est, ref.k_est)
    assert torch.equal(out.rates, ref.rates)


def test_in_order_arsvd_equals_speculative(cuda):
    """spec_passes = 0 (in-order from the first step) and the default policy give
    the same trajectory, and both match the reference golden at eta = 0.9."""
    g = load_golden("traj_C2s")
    spec = S.C2
    H = torch.from_numpy(S.channels(spec, trials=[0, 1], t1=24)).to(cuda)
    noise = torch.full((2, spec.K), spec.noise_var, dtype=torch.float64, device=cuda)
    outs = []
    for sp in (0, 2):
        cfg = TrajectoryConfig(alpha=spec.alpha, eta=0.9, k_init=spec.k_init, p=spec.p,
                               i_max=spec.i_max, spec_passes=sp)
        rn = TrajectoryRunner(2, spec.K, spec.N, torch.complex128, cfg, cuda)
        st = OmegaStreams.for_method(0, 0.9, [0, 1])
        om = torch.from_numpy(st.window(24 * rn.normals_per_step_max())).to(cuda)
        outs.append(rn.run_chunk(H, noise, om))
    a, b = outs
    assert torch.equal(a.k_est, b.k_est) and torch.equal(a.method, b.method)
    assert torch.equal(a.consumed, b.consumed)
    for t in (0, 1):
        assert np.array_equal(a.k_est[t].cpu().numpy(), g[f"t{t}_e900_k_est"])
        np.testing.assert_allclose(a.rates[t].cpu().numpy(), g[f"t{t}_e900_rates"], rtol=1e-10)


def test_per_row_eta_equals_separate_runners(cuda):
    spec = S.C2.with_(B=3, T=30)
    trials = [0, 1, 2]
    H, noise, _ = _setup(cuda, spec, None, trials)
    etas = (0.9, 0.8)
    sep = []
    for eta in etas:
        cfg = TrajectoryConfig(alpha=spec.alpha, eta=eta, k_init=spec.k_init, p=spec.p,
                               i_max=spec.i_max)
        rn = TrajectoryRunner(3, spec.K, spec.N, torch.complex128, cfg, cuda)
        st = DeviceOmegaStreams.for_method(spec.seed, eta, trials, cuda)
        sep.append(rn.run_chunk(H, noise, st.window(spec.T * rn.normals_per_step_max())))
    cfg = TrajectoryConfig(alpha=spec.alpha, eta=[e for e in etas for _ in trials],
                           k_init=spec.k_init, p=spec.p, i_max=spec.i_max)
    rn = TrajectoryRunner(6, spec.K, spec.N, torch.complex128, cfg, cuda)
    gens = [np.random.default_rng(S.stream_seed(spec.seed, S.method_label(e), t))
            for e in etas for t in trials]
    st = DeviceOmegaStreams(gens, cuda)
    both = rn.run_chunk(H.repeat(2, 1, 1, 1), noise.repeat(2, 1),
                        st.window(spec.T * rn.normals_per_step_max()))
    for i in range(2):
        assert torch.equal(both.k_est[3 * i:3 * i + 3], sep[i].k_est)
        assert torch.equal(both.method[3 * i:3 * i + 3], sep[i].method)
        assert torch.equal(both.rates[3 * i:3 * i + 3], sep[i].rates)


def test_rng_locate_matches_host_stream(cuda):
    """Advancing by the located raw offsets lands each stream exactly where
    numpy's Generator is after drawing the same number of normals."""
    trials = [0, 3, 7]
    dev = DeviceOmegaStreams.for_method(0, 0.9, trials, cuda)
    host = OmegaStreams.for_method(0, 0.9, trials)
    for L, used in [(4000, [0, 1, 3999]), (30000, [12345, 29999, 7]), (5000, [5000, 2500, 1])]:
        d = dev.window(L).cpu().numpy()
        h = host.window(L)
        assert (d == h).mean() > 0.999
        dev.advance(used)
        host.advance(used)
    d = dev.window(1000).cpu().numpy()
    assert (d == host.window(1000)).mean() > 0.999


@pytest.mark.parametrize("rounds,T,eta", [(-1, 200, 0.9), (1, 200, 0.9), (2, 120, 0.8), (0, 60, 0.9)])
def test_screen_rounds_settle_the_cursors(cuda, rounds, T, eta):
    """Screen-only cursor-resolution rounds (lrz_arsvd want_factor 2 + lrz_spec_verify,
    then the in-order warp walk for what is left) against the in-order exact
    trajectory on full-length Woodbury-regime C2 trials: iteration counts,
    consumption, ranks, methods identical; settled in one exact pass."""
    spec = S.C2.with_(B=4, T=T)
    trials = list(range(4))
    H, noise, _ = _setup(cuda, spec, None, trials)
    outs = []
    for sp, r in ((0, 0), (2, rounds)):
        cfg = TrajectoryConfig(alpha=spec.alpha, eta=eta, k_init=spec.k_init, p=spec.p,
                               i_max=spec.i_max, spec_passes=sp, walk_first=True,
                               screen_rounds=r)
        rn = TrajectoryRunner(4, spec.K, spec.N, torch.complex128, cfg, cuda)
        st = DeviceOmegaStreams.for_method(spec.seed, eta, trials, cuda)
        outs.append(rn.run_chunk(H, noise, st.window(spec.T * rn.normals_per_step_max())))
    a, b = outs
    assert torch.equal(a.iters, b.iters) and torch.equal(a.consumed, b.consumed)
    assert torch.equal(a.k_est, b.k_est) and torch.equal(a.method, b.method)
    assert b.spec_passes == 1
    torch.testing.assert_close(a.rates, b.rates, rtol=1e-10, atol=0)


@pytest.mark.parametrize("walk_first", [True, False])
def test_cursor_walk_equals_in_order(cuda, walk_first):
    """The energy-screen cursor walk (lrz_arsvd_walk) followed by one speculative
    pass gives the in-order trajectory (iteration counts, consumption, ranks,
    methods, rates) on a Woodbury-regime C2 slice (eta = 0.9)."""
    spec = S.C2.with_(B=6, T=40)
    trials = list(range(6))
    H, noise, _ = _setup(cuda, spec, None, trials)
    outs = []
    for sp, wf in ((0, None), (2, walk_first)):
        cfg = TrajectoryConfig(alpha=spec.alpha, eta=0.9, k_init=spec.k_init, p=spec.p,
                               i_max=spec.i_max, spec_passes=sp, walk_first=wf)
        rn = TrajectoryRunner(6, spec.K, spec.N, torch.complex128, cfg, cuda)
        st = DeviceOmegaStreams.for_method(spec.seed, 0.9, trials, cuda)
        outs.append(rn.run_chunk(H, noise, st.window(spec.T * rn.normals_per_step_max())))
    a, b = outs
    assert (a.method.cpu().numpy() == 1).mean() > 0.5          # Woodbury regime
    assert torch.equal(a.iters, b.iters) and torch.equal(a.consumed, b.consumed)
    assert torch.equal(a.k_est, b.k_est) and torch.equal(a.method, b.method)
    assert b.spec_passes <= 2
    torch.testing.assert_close(a.rates, b.rates, rtol=1e-10, atol=0)


@pytest.mark.parametrize("name,B,T,chunk,dtype", [("C2", 6, 48, 16, "c128"),
                                                   ("C3", 4, 24, 8, "c64")])
@pytest.mark.parametrize("schedule", ["back", "heavy"])
def test_two_stream_schedules_equal_the_synchronous_runner(cuda, name, B, T, chunk, dtype,
                                                           schedule):
    """run_chunk(sync=False) with back_stream (chunk c's chain / precoder beside
    chunk c + 1's front stages) and with heavy_stream + gram_async (Grams and
    precoder products on a low-priority stream) reproduce the synchronous pass
    bit for bit over several chunks, with zero verifier flags."""
    spec = S.CONFIGS[name].with_(B=B, T=T, dtype=dtype)
    trials = list(range(B))
    tdt = torch.complex64 if dtype == "c64" else torch.complex128
    H, noise, cfg = _setup(cuda, spec, spec.eta, trials)
    H = H.to(tdt)
    chunks = [H[:, t0:t0 + chunk].contiguous() for t0 in range(0, T, chunk)]
    st = DeviceOmegaStreams.for_method(spec.seed, spec.eta, trials, cuda)
    cur = torch.cuda.current_stream(cuda)

    def run(mode):
        rn = TrajectoryRunner(B, spec.K, spec.N, tdt, cfg, cuda)
        st.raw.zero_()
        st.consumed_total.zero_()
        outs, flags = [], torch.zeros(2, dtype=torch.int32, device=cuda)
        if mode == "heavy":
            heavy = torch.cuda.Stream(cuda, priority=0)
            light = torch.cuda.Stream(cuda, priority=-1)
            light.wait_stream(cur)
            with torch.cuda.stream(light):
                g = rn.gram_async(chunks[0], heavy)
                for i, Hc in enumerate(chunks):
                    g_next = rn.gram_async(chunks[i + 1], heavy) if i + 1 < len(chunks) else None
                    om = st.window(chunk * rn.normals_per_step_max())
                    r = rn.run_chunk(Hc, noise, om, sync=False, heavy_stream=heavy, gram=g,
                                     keep_A_inv=True)
                    flags.add_(r.flags)
                    st.advance(r.consumed)
                    outs.append(r)
                    g = g_next
            cur.wait_stream(light)
            cur.wait_stream(heavy)
        else:
            back = torch.cuda.Stream(cuda, priority=-1) if mode == "back" else None
            for Hc in chunks:
                om = st.window(chunk * rn.normals_per_step_max())
                r = rn.run_chunk(Hc, noise, om, sync=back is None, back_stream=back,
                                 keep_A_inv=True)
                if r.flags is not None:
                    flags.add_(r.flags)
                st.advance(r.consumed)
                outs.append(r)
            if back is not None:
                cur.wait_stream(back)
        torch.cuda.synchronize()
        assert int(flags.abs().sum()) == 0
        return outs

    ref = run("sync")
    got = run(schedule)
    for a, b in zip(ref, got):
        assert torch.equal(a.method, b.method) and torch.equal(a.k_est, b.k_est)
        assert torch.equal(a.iters, b.iters) and torch.equal(a.consumed, b.consumed)
        assert torch.equal(a.rates, b.rates) and torch.equal(a.info, b.info)
        assert torch.equal(a.A_inv, b.A_inv)
