"""The large BASELINE configs at their full trial counts (C3: 256 trials x 500
steps, C4: 1024 trials, C5: 64 trials x 100 steps) through the
everything-on-device campaign: size-independent properties (chunking
invariance, finite positive rates, the dispatcher's rank rule) plus an
oracle replay of the first steps of trial 0 (full sizes are
checked through properties, small prefixes against the oracle)."""

import numpy as np
import pytest

from oracle import port, sweep
from paper_2512_16543_b200 import scenario as S
from paper_2512_16543_b200.trajectory import run_campaign_device

pytestmark = pytest.mark.gpu


def _replay(spec, eta, steps):
    H = S.trial_channels(spec, 0, 0, steps).astype(np.complex64)
    sk = np.random.default_rng(S.stream_seed(spec.seed, S.method_label(eta), 0))
    return sweep.sweep_trial(H, spec.alpha, S.noise_vector(spec), 1.0,
                             port.Cfg(eta, spec.k_init, spec.p, spec.i_max), sk)


@pytest.mark.parametrize("name,T,chunks,steps", [
    ("C3", 500, (50, 125), 12),
    ("C4", 24, (8, 12), 6),
    ("C5", 100, (10, 25), 4),
])
def test_full_trial_count_properties_and_oracle_prefix(cuda, name, T, chunks, steps):
    spec = S.CONFIGS[name].with_(T=T)
    eta = spec.eta
    a = run_campaign_device(spec, eta, range(spec.B), cuda, chunk=chunks[0])
    b = run_campaign_device(spec, eta, range(spec.B), cuda, chunk=chunks[1])
    assert np.array_equal(a.method, b.method) and np.array_equal(a.k_est, b.k_est)
    np.testing.assert_allclose(a.rates, b.rates, rtol=1e-12)
    assert np.all(np.isfinite(a.rates)) and np.all(a.rates > 0)
    m, k = a.method[:, 1:], a.k_est[:, 1:]
    # dispatcher rule (lowrank.py:345-359): none iff k_est == 0; Woodbury only
    # when 0 < k_est <= K/2 (full otherwise, or when the aux matrix is singular)
    assert np.array_equal(m == 2, k == 0)
    assert np.all((k[m == 1] > 0) & (2 * k[m == 1] <= spec.K))
    assert np.all(a.method[:, 0] == 0)
    ref = _replay(spec, eta, steps)
    tie = ref.margin < 1e-6
    ok = (a.k_est[0, :steps] == ref.k_est) | tie
    assert ok.all(), (a.k_est[0, :steps], ref.k_est)
    if (a.k_est[0, :steps] == ref.k_est).all():
        assert np.array_equal(a.method[0, :steps], ref.method)
        np.testing.assert_allclose(a.rates[0, :steps], ref.rates, rtol=1e-4)
