"""Host side of the LEO campaign (no GPU): scenario mirror, user drop, DFT
factors, against the oracle and the reference golden constants."""

import math

import numpy as np
import pytest

from oracle import leo as OL
from paper_2512_16543_b200 import leo as L
from paper_2512_16543_b200.errors import RangeError

from conftest import load_golden
from test_oracle_leo import cfg_from


@pytest.mark.parametrize("name", ["leo_small", "leo_rect", "leo_default", "leo_full_trial"])
def test_scenario_constants(name):
    g = load_golden(name)
    cfg = cfg_from(g) if name != "leo_full_trial" else L.ScenarioConfig().validate()
    assert cfg.resolved_alpha == float(g["alpha"])
    assert cfg.noise_variance_W == float(g["noise"])


def test_validate_ranges():
    for kw in (dict(K=0), dict(N_RF=8), dict(eta_list=()), dict(eta_list=(1.5,)),
               dict(pass_s=1.01, update_rate_Hz=7.0), dict(beam_hold=0), dict(n_reset=-1)):
        with pytest.raises(RangeError):
            L.ScenarioConfig(**kw).validate()


def test_user_drop_matches_oracle():
    cfg = L.ScenarioConfig().validate()
    for trial in (0, 3):
        a = L.place_users(cfg, np.random.default_rng(L.stream_seed(0, "channel", trial)))
        b = OL.ut_positions(cfg, np.random.default_rng(OL.seed_seq(0, "channel", trial)))
        assert np.array_equal(a[:, :3], b)
        assert np.all(a[:, 3] == cfg.ut_gain_dBi)
        assert np.all(a[:, 4] == min(10 ** (cfg.K_R_dB / 10), 1e12))


def test_dft_factors_kron_is_the_codebook():
    f = L.dft_factors(4, 8)
    Dx, Dy = f[:16].reshape(4, 4), f[16:].reshape(8, 8)
    assert np.array_equal(np.kron(Dx, Dy), OL.codebook(4, 8))


def test_leo_cfg_fields():
    cfg = L.ScenarioConfig().validate()
    c = L.leo_cfg(cfg)
    assert c.K == 16 and c.N_RF == 16 and c.n_x == 16
    assert math.isclose(c.orbit_rate * c.orbit_radius, 7560.0, abs_tol=10.0)
    assert c.dt == 0.05 and c.nlos_block == 1 and c.beam_hold == 1
