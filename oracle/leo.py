"""CPU restatement of the reference's LEO pass simulator, hybrid beam
selection and Monte-Carlo campaign (TEST INFRASTRUCTURE: only tests/,
``__graft_entry__.smoke()`` and bench CPU legs import this module; the
product path never does).

Follows, step for step:

* pass geometry -- ``channel.py:236-289`` (circular equatorial orbit,
  nadir-pointing frame with x along-track, elevation mask);
* user placement -- ``channel.py:292-311`` and ``UserTerminal.position_ecef``
  ``channel.py:73-83`` (disk of ``footprint_radius_m``, spherical Earth);
* conjugated manifold rows -- ``channel.py:128-137``;
* 2-D DFT codebook / beam powers / greedy selection -- ``channel.py:176-233``;
* snapshot assembly -- ``channel.py:352-384`` and ``draw_nlos`` ``:387-392``;
* the per-trial method sweep -- ``harness._sweep_trial`` ``harness.py:188-257``;
* the campaign reduction -- ``harness.run_campaign`` ``harness.py:313-383``
  and ``ecdf`` ``harness.py:95-104``.

Pinned against fixtures produced by the reference itself
(tests/golden/gen_golden_leo.py -> tests/golden/leo_*.npz).
"""

from __future__ import annotations

import math
import zlib
from dataclasses import dataclass, field

import numpy as np

from . import port

R_EARTH = 6371e3                 # channel.py:24
GM = 3.986004418e14              # channel.py:25
C_LIGHT = 299_792_458.0          # channel.py:26
K_BOLTZ = 1.380649e-23           # channel.py:27
T_NOISE = 290.0                  # channel.py:28
KR_CAP = 1e12                    # channel.py:29
DECISION = {"full": 0, "woodbury": 1, "none": 2}


class OracleBelowMask(Exception):
    """BelowMinElevationError analogue (channel.py:280-284)."""


def label_of(eta):
    return "conventional" if eta is None else f"wb_arsvd_eta{eta:g}"


def seed_seq(master, label, trial):
    return np.random.SeedSequence([int(master), zlib.crc32(label.encode("utf-8")), int(trial)])


# -- scenario-derived scalars (config.py:63-91) -------------------------------------

def wavelength(cfg):
    return C_LIGHT / cfg.carrier_Hz


def noise_w(cfg):
    return K_BOLTZ * T_NOISE * cfg.bandwidth_Hz


def alpha_of(cfg):
    if cfg.alpha is not None:
        return cfg.alpha
    lam = wavelength(cfg)
    fs = 20.0 * math.log10(4.0 * math.pi * cfg.altitude_m / lam)
    g = 10.0 ** ((cfg.ut_gain_dBi - fs - cfg.atmospheric_loss_dB) / 20.0)
    return cfg.K * (noise_w(cfg) / g ** 2) / cfg.P_t_W


def n_steps(cfg):
    return int(round(cfg.pass_s * cfg.update_rate_Hz))


# -- pass context ---------------------------------------------------------------------

@dataclass
class Pass:
    cfg: object
    ut_xyz: np.ndarray        # (K, 3) ECEF
    gain_dbi: np.ndarray      # (K,)
    k_lin: np.ndarray         # (K,)
    elem: np.ndarray          # (N, 3) element positions, metres
    codebook: np.ndarray      # (N, N)
    lam: float


def elements(cfg, lam):
    d = cfg.spacing_wavelengths * lam
    gx, gy = np.meshgrid(np.arange(cfg.n_x), np.arange(cfg.n_y), indexing="ij")
    out = np.zeros((cfg.n_x * cfg.n_y, 3))
    out[:, 0] = (gx.ravel() - (cfg.n_x - 1) / 2.0) * d
    out[:, 1] = (gy.ravel() - (cfg.n_y - 1) / 2.0) * d
    return out


def codebook(n_x, n_y):
    def f(n):
        i = np.arange(n)
        return np.exp(-2j * np.pi * np.outer(i, i) / n) / math.sqrt(n)
    return np.kron(f(n_x), f(n_y))


def ut_positions(cfg, rng):
    """Uniform disk drop; positions via per-UT scalar math like
    UserTerminal.position_ecef (channel.py:73-83, 292-311)."""
    K = cfg.K
    rad = cfg.footprint_radius_m * np.sqrt(rng.random(K))
    brg = 2.0 * np.pi * rng.random(K)
    lat = np.degrees((rad * np.cos(brg)) / R_EARTH)
    lon = np.degrees((rad * np.sin(brg)) / R_EARTH)
    xyz = np.empty((K, 3))
    for n in range(K):
        a, b = math.radians(float(lat[n])), math.radians(float(lon[n]))
        xyz[n] = [R_EARTH * math.cos(a) * math.cos(b), R_EARTH * math.cos(a) * math.sin(b),
                  R_EARTH * math.sin(a)]
    return xyz


def make_pass(cfg, rng) -> Pass:
    lam = wavelength(cfg)
    xyz = ut_positions(cfg, rng)
    K = cfg.K
    return Pass(cfg, xyz, np.full(K, float(cfg.ut_gain_dBi)),
                np.minimum(10.0 ** (np.full(K, float(cfg.K_R_dB)) / 10.0), KR_CAP),
                elements(cfg, lam), codebook(cfg.n_x, cfg.n_y), lam)


def orbit(cfg, xyz, t):
    """(theta, phi, slant) at pass time t (channel.py:242-289)."""
    if not 0.0 <= t <= cfg.pass_s:
        raise ValueError(f"t={t} outside the pass")
    R = R_EARTH + cfg.altitude_m
    ang = math.sqrt(GM / R ** 3) * (t - cfg.pass_s / 2.0)
    sat = R * np.array([math.cos(ang), math.sin(ang), 0.0])
    xb = np.array([-math.sin(ang), math.cos(ang), 0.0])
    zb = -sat / R
    yb = np.cross(zb, xb)
    dv = xyz - sat
    rng_m = np.linalg.norm(dv, axis=1)
    u = (dv / rng_m[:, None]) @ np.stack([xb, yb, zb], axis=1)
    theta = np.arccos(np.clip(u[:, 2], -1.0, 1.0))
    phi = np.arctan2(u[:, 1], u[:, 0])
    pn = np.linalg.norm(xyz, axis=1)
    s_el = np.einsum("ij,ij->i", xyz / pn[:, None], -dv) / rng_m
    el = np.arcsin(np.clip(s_el, -1.0, 1.0))
    if np.any(el < math.radians(cfg.min_elevation_deg)):
        raise OracleBelowMask(f"elevation {math.degrees(el.min()):.2f} deg at t={t}")
    return theta, phi, rng_m


def manifold(theta, phi, elem, lam):
    st = np.sin(theta)
    kv = (2.0 * np.pi / lam) * np.stack([st * np.cos(phi), st * np.sin(phi), np.cos(theta)],
                                        axis=1)
    return np.exp(-1j * (kv @ elem.T)) / math.sqrt(elem.shape[0])


def beam_powers(Ht, n_x, n_y):
    sp = np.fft.fft2(Ht.reshape(Ht.shape[0], n_x, n_y), norm="ortho")
    return np.abs(sp.reshape(Ht.shape[0], -1)) ** 2


def pick_beams(power, N_RF):
    """Greedy per-UT best unused codeword, stable ties to the lowest index,
    then fill by best-over-UTs power (channel.py:202-233).  Returns indices."""
    K, n_cb = power.shape
    if not K <= N_RF <= n_cb:
        raise ValueError("need K <= N_RF <= codebook size")
    taken = np.zeros(n_cb, bool)
    cols = []
    for n in range(K):
        for j in np.argsort(-power[n], kind="stable"):
            if not taken[j]:
                taken[j] = True
                cols.append(int(j))
                break
    if len(cols) < N_RF:
        for j in np.argsort(-power.max(axis=0), kind="stable"):
            if len(cols) == N_RF:
                break
            if not taken[j]:
                taken[j] = True
                cols.append(int(j))
    return np.array(cols, dtype=np.int64)


def nlos_draw(cfg, rng):
    shp = (cfg.K, cfg.n_x * cfg.n_y)
    return math.sqrt(0.5) * (rng.standard_normal(shp) + 1j * rng.standard_normal(shp))


@dataclass
class Snap:
    H: np.ndarray
    H_tilde: np.ndarray
    cols: np.ndarray
    F_RF: np.ndarray
    H_eff: np.ndarray


def snapshot(ps: Pass, t, nlos, cols=None) -> Snap:
    """channel.py:352-384 with the NLOS draw passed in and beams by index."""
    cfg = ps.cfg
    theta, phi, slant = orbit(cfg, ps.ut_xyz, t)
    Ht = manifold(theta, phi, ps.elem, ps.lam)
    fs = 20.0 * np.log10(4.0 * np.pi * slant / ps.lam)
    g = 10.0 ** ((ps.gain_dbi - fs - cfg.atmospheric_loss_dB) / 20.0)
    nt = ps.elem.shape[0]
    H = (np.sqrt(ps.k_lin / (ps.k_lin + 1.0))[:, None] * (g[:, None] * Ht)
         + np.sqrt(1.0 / (ps.k_lin + 1.0))[:, None] * ((g / math.sqrt(nt))[:, None] * nlos))
    if cols is None:
        cols = pick_beams(beam_powers(Ht, cfg.n_x, cfg.n_y), cfg.N_RF)
    F = ps.codebook[:, cols]
    return Snap(H, Ht, cols, F, Ht @ F)


# -- the sweep (harness.py:188-257) -----------------------------------------------------

@dataclass
class Run:
    label: str
    eta: float | None
    rng: np.random.Generator
    cfg: port.Cfg | None
    state: port.State | None = None
    rates: list = field(default_factory=list)
    methods: list = field(default_factory=list)
    k_est: list = field(default_factory=list)
    costs: list = field(default_factory=list)
    total_cost: float = 0.0
    k_sum: int = 0
    k_count: int = 0
    counts: dict = field(default_factory=lambda: {"full": 0, "woodbury": 0, "none": 0})


def sweep_trial(cfg, specs, trial, master_seed, sketch_labels=None, keep_snaps=None,
                steps=None):
    """specs: list of (label, eta-or-None).  Returns label -> Run.  keep_snaps:
    optional list receiving (H_eff, H @ F_RF, cols) per step; steps: stop
    after this many snapshots (a prefix of the pass)."""
    crng = np.random.default_rng(seed_seq(master_seed, "channel", trial))
    ps = make_pass(cfg, crng)
    noise = np.full(cfg.K, noise_w(cfg))
    alpha = alpha_of(cfg)
    K = cfg.K
    runs = []
    for label, eta in specs:
        sl = (sketch_labels or {}).get(label, label)
        runs.append(Run(label, eta, np.random.default_rng(seed_seq(master_seed, sl, trial)),
                        None if eta is None else port.Cfg(eta, cfg.k_init, cfg.p, cfg.i_max)))
    dt = 1.0 / cfg.update_rate_Hz
    prev = cols = nl = None
    for i in range(n_steps(cfg) if steps is None else min(steps, n_steps(cfg))):
        if i % cfg.nlos_block_len == 0:
            nl = nlos_draw(cfg, crng)
        sn = snapshot(ps, i * dt, nl, cols if i % cfg.beam_hold != 0 else None)
        cols = sn.cols
        if keep_snaps is not None:
            keep_snaps.append((sn.H_eff, sn.H @ sn.F_RF, sn.cols))
        for r in runs:
            if r.eta is None or r.state is None or (cfg.n_reset > 0 and i % cfg.n_reset == 0):
                r.state = port.gram_matrix(sn.H_eff, alpha)
                m, k, c = "full", 0, port.cost_full(K)
            else:
                r.state, m, k, c, _ = port.update_inverse(r.state, prev, sn.H_eff - prev,
                                                          r.cfg, r.rng)
                r.k_sum += k
                r.k_count += 1
            F_BB, _ = port.rzf_precoder(sn.H_eff, r.state.A_inv, sn.F_RF, cfg.P_t_W)
            _, tot, _ = port.sum_rate(sn.H, sn.F_RF, F_BB, noise)
            r.rates.append(tot)
            r.methods.append(DECISION[m])
            r.k_est.append(k)
            r.costs.append(c)
            r.total_cost += c
            r.counts[m] += 1
        prev = sn.H_eff
    return {r.label: r for r in runs}


def ecdf(samples):
    x = np.sort(np.asarray(samples, dtype=float).ravel())
    if x.size == 0:
        raise ValueError("empty")
    v = np.unique(x)
    return np.column_stack([v, np.searchsorted(x, v, side="right") / x.size])


def campaign(cfg, master_seed=None):
    """harness.run_campaign reduction over mc_runs trials (serial)."""
    seed = cfg.seed if master_seed is None else master_seed
    etas = sorted(set(cfg.eta_list), reverse=True)
    specs = [(label_of(None), None)] + [(label_of(e), e) for e in etas]
    per = [sweep_trial(cfg, specs, i, seed) for i in range(cfg.mc_runs)]
    out = {"labels": [s[0] for s in specs], "pooled": {}, "trial_means": {}, "mean_rate": {},
           "mean_cost": {}, "mean_k": {}, "counts": {}, "decisions": {}}
    for lab, _ in specs:
        pooled = np.concatenate([np.array(p[lab].rates) for p in per])
        out["pooled"][lab] = pooled
        out["trial_means"][lab] = np.array([np.mean(p[lab].rates) for p in per])
        out["mean_rate"][lab] = float(pooled.mean())
        out["mean_cost"][lab] = float(np.mean([p[lab].total_cost for p in per]))
        ks = sum(p[lab].k_sum for p in per)
        kc = sum(p[lab].k_count for p in per)
        out["mean_k"][lab] = ks / kc if kc else 0.0
        cnt = {"full": 0, "woodbury": 0, "none": 0}
        for p in per:
            for key, v in p[lab].counts.items():
                cnt[key] += v
        out["counts"][lab] = cnt
        out["decisions"][lab] = [np.array(p[lab].methods, np.uint8) for p in per]
    conv = label_of(None)
    out["table"] = [(conv, None, 0.0, 0.0)] + [
        (label_of(e), e, 100.0 * (1.0 - out["mean_cost"][label_of(e)] / out["mean_cost"][conv]),
         100.0 * (1.0 - out["mean_rate"][label_of(e)] / out["mean_rate"][conv])) for e in etas]
    return out
