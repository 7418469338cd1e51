"""Device sketch streams vs numpy's Generator(PCG64).standard_normal."""

import numpy as np
import pytest
import torch

from paper_2512_16543_b200 import scenario as S
from paper_2512_16543_b200.omega import DeviceOmegaStreams, OmegaStreams

pytestmark = pytest.mark.gpu


def test_device_normals_match_numpy(cuda):
    trials = [0, 1, 5, 63]
    dev = DeviceOmegaStreams.for_method(0, 0.999, trials, cuda)
    host = OmegaStreams.for_method(0, 0.999, trials)
    for L, used in [(50000, [3200, 0, 12345, 49999]), (70000, [7, 7, 7, 7]), (1000, [1000] * 4),
                    (1_500_000, [1_499_999, 3, 700_000, 1])]:  # ~1,700 tail values
        d = dev.window(L).cpu().numpy()
        h = host.window(L)
        assert int(dev._status.sum().item()) == 0
        # bit-exact, ziggurat tail included (glibc-compatible log1p on the device)
        assert np.array_equal(d.view(np.uint64), h.view(np.uint64)), int((d != h).sum())
        dev.advance(used)
        host.advance(used)
    assert np.array_equal(dev.consumed_total.cpu().numpy(), host.consumed_total)


def test_device_streams_drive_the_runner(cuda):
    """A C2-sample trajectory with device sketches equals the reference golden."""
    from conftest import load_golden
    from paper_2512_16543_b200 import TrajectoryConfig, TrajectoryRunner
    g = load_golden("traj_C2s")
    spec = S.C2
    H = torch.from_numpy(S.channels(spec, trials=[0, 1], t1=24)).to(cuda)
    cfg = TrajectoryConfig(alpha=spec.alpha, eta=0.9, k_init=spec.k_init, p=spec.p,
                           i_max=spec.i_max)
    rn = TrajectoryRunner(2, spec.K, spec.N, torch.complex128, cfg, cuda)
    st = DeviceOmegaStreams.for_method(0, 0.9, [0, 1], cuda)
    noise = torch.full((2, spec.K), spec.noise_var, dtype=torch.float64, device=cuda)
    ks, rates = [], []
    for t0 in (0, 10):
        t1 = 10 if t0 == 0 else 24
        om = st.window((t1 - t0) * rn.normals_per_step_max())
        r = rn.run_chunk(H[:, t0:t1].contiguous(), noise, om)
        st.advance(r.consumed)
        ks.append(r.k_est.cpu().numpy())
        rates.append(r.rates.cpu().numpy())
    k = np.concatenate(ks, 1)
    rt = np.concatenate(rates, 1)
    for b in (0, 1):
        assert np.array_equal(k[b], g[f"t{b}_e900_k_est"])
        assert np.allclose(rt[b], g[f"t{b}_e900_rates"], rtol=1e-10)


@pytest.mark.parametrize("name,dtype", [("C1", "c128"), ("C2", "c128"), ("C3", "c64")])
def test_device_channels_match_host(cuda, name, dtype):
    spec = S.CONFIGS[name].with_(dtype=dtype, B=3, T=7)
    dc = S.DeviceChannels(spec, [0, 1, 2], cuda)
    Hd = dc.generate(2, 7).cpu().numpy()
    Hh = S.channels(spec, trials=[0, 1, 2], t0=2, t1=7)
    err = np.abs(Hd - Hh).max() / np.abs(Hh).max()
    assert err < (1e-13 if dtype == "c128" else 1e-6), err


def test_device_channels_drive_golden_trajectory(cuda):
    from conftest import load_golden
    from paper_2512_16543_b200 import TrajectoryConfig, run_trajectory
    g = load_golden("traj_C2s")
    spec = S.C2.with_(B=2, T=24)
    H = S.DeviceChannels(spec, [0, 1], cuda).generate(0, 24)
    cfg = TrajectoryConfig(alpha=spec.alpha, eta=0.9, k_init=spec.k_init, p=spec.p,
                           i_max=spec.i_max)
    res = run_trajectory(H, S.noise_vector(spec), cfg,
                         DeviceOmegaStreams.for_method(0, 0.9, [0, 1], cuda))
    for b in (0, 1):
        assert np.array_equal(res.k_est[b], g[f"t{b}_e900_k_est"])
        assert np.allclose(res.rates[b], g[f"t{b}_e900_rates"], rtol=1e-10)


def test_campaign_device_chunked_matches_host_path(cuda):
    """Everything-on-device campaign (synthesised channels, device sketches,
    time chunks) equals the host-input runner on the same trials."""
    from paper_2512_16543_b200 import TrajectoryConfig, run_trajectory
    from paper_2512_16543_b200.trajectory import run_campaign_device
    spec = S.C2.with_(B=3, T=30)
    dev_res = run_campaign_device(spec, 0.9, [0, 1, 2], cuda, chunk=11)
    H = S.channels(spec, trials=[0, 1, 2])
    cfg = TrajectoryConfig(alpha=spec.alpha, eta=0.9, k_init=spec.k_init, p=spec.p,
                           i_max=spec.i_max)
    host_res = run_trajectory(H, S.noise_vector(spec), cfg,
                              OmegaStreams.for_method(0, 0.9, [0, 1, 2]))
    assert np.array_equal(dev_res.k_est, host_res.k_est)
    assert np.array_equal(dev_res.method, host_res.method)
    assert np.allclose(dev_res.rates, host_res.rates, rtol=1e-10)
