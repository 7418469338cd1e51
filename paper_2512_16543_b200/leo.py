"""The reference's own LEO Monte-Carlo campaign on the GPU (SURVEY.md 8(f)
"next" #3 hybrid F_RF path and #4 campaign reduction).

Drop-in for the campaign surface of ``leorzf.harness`` (harness.py:64-104,
259-383) over the scenario of ``leorzf.config.ScenarioConfig``
(config.py:27-91): same names, same per-(method, trial) random streams, same
decisions and accounting.  What runs where:

* host: per trial, the user drop from the channel stream (2 K uniforms,
  channel.py:292-311) -- then the stream's PCG64 state moves to the device;
* device, per (trial, step) (``lrz_leo_snapshot``): orbit geometry, manifold
  rows, Rician channel with the NLOS block drawn by the device RNG from the
  same channel stream, DFT beam powers, greedy beam selection (held for
  ``beam_hold`` steps) and the products H~ F_RF / H F_RF;
* device, per method: the batched trajectory runner (Gram, gram_delta,
  speculative arSVD, dispatcher, Woodbury chain) on H_eff, then the hybrid
  precoder / rate (``lrz_hybrid_precode_rate``) and the per-trial cost / rank /
  decision totals (``lrz_campaign_reduce``);
* host: pooled means, the comparison table and the ECDF over the per-step
  rates, as ``run_campaign`` does (harness.py:336-383).

All methods of a trial see the same channel (it is generated once per chunk
and shared), and trials shard across ranks with one gather at the end.
"""

from __future__ import annotations

import math
import zlib
from dataclasses import dataclass, field, replace

import numpy as np
import torch

from . import _native as Nn
from . import ops
from .errors import (BelowMinElevationError, EmptyInputError, RangeError, SingularMatrixError,
                     ZeroPrecoderError)
from .lowrank import cost_full, cost_wb_arsvd
from .omega import DeviceOmegaStreams
from .trajectory import TrajectoryConfig, TrajectoryRunner, step_costs

EARTH_RADIUS_M = 6371e3          # channel.py:24
GM_EARTH = 3.986004418e14        # channel.py:25
SPEED_OF_LIGHT_M_S = 299_792_458.0
BOLTZMANN_J_K = 1.380649e-23
SYSTEM_NOISE_TEMP_K = 290.0
RICIAN_K_CAP = 1e12
CHANNEL_STREAM = "channel"
DECISION_CODES = {"full": 0, "woodbury": 1, "none": 2}   # harness.py:29
_METHOD_NAMES = ("full", "woodbury", "none")


@dataclass
class ScenarioConfig:
    """Scenario of one campaign; same fields, defaults and derived values as
    the reference's ``ScenarioConfig`` (config.py:27-91), so either object
    can be passed to the functions below."""

    carrier_Hz: float = 18e9
    altitude_m: float = 600e3
    n_x: int = 16
    n_y: int = 16
    spacing_wavelengths: float = 0.5
    N_RF: int = 16
    P_t_W: float = 100.0
    ut_gain_dBi: float = 39.7
    K: int = 16
    K_R_dB: float = 10.0
    pass_s: float = 120.0
    update_rate_Hz: float = 20.0
    mc_runs: int = 50
    eta_list: tuple = (0.9, 0.8, 0.65)
    k_init: int = 2
    p: int = 1
    i_max: int = 8
    footprint_radius_m: float = 225e3
    bandwidth_Hz: float = 50e6
    min_elevation_deg: float = 10.0
    atmospheric_loss_dB: float = 0.0
    alpha: float | None = None
    n_reset: int = 1200
    nlos_block_len: int = 1
    beam_hold: int = 1
    seed: int = 0

    @property
    def n_elements(self) -> int:
        return self.n_x * self.n_y

    @property
    def noise_variance_W(self) -> float:
        return BOLTZMANN_J_K * SYSTEM_NOISE_TEMP_K * self.bandwidth_Hz

    @property
    def reference_gain(self) -> float:
        lam = SPEED_OF_LIGHT_M_S / self.carrier_Hz
        fspl = 20.0 * math.log10(4.0 * math.pi * self.altitude_m / lam)
        return 10.0 ** ((self.ut_gain_dBi - fspl - self.atmospheric_loss_dB) / 20.0)

    @property
    def resolved_alpha(self) -> float:
        if self.alpha is not None:
            return self.alpha
        return self.K * (self.noise_variance_W / self.reference_gain ** 2) / self.P_t_W

    @property
    def n_snapshots(self) -> int:
        return int(round(self.pass_s * self.update_rate_Hz))

    def validate(self) -> "ScenarioConfig":
        """Range checks of config.py:93-135 (RangeError)."""
        chk = [
            (self.K >= 1, f"K must be >= 1, got {self.K}"),
            (self.K <= self.N_RF <= self.n_elements,
             f"need K <= N_RF <= N_t, got K={self.K}, N_RF={self.N_RF}, N_t={self.n_elements}"),
            (self.n_x >= 1 and self.n_y >= 1, "array dimensions must be >= 1"),
        ]
        for name in ("carrier_Hz", "altitude_m", "spacing_wavelengths", "P_t_W", "pass_s",
                     "update_rate_Hz", "bandwidth_Hz"):
            chk.append((getattr(self, name) > 0, f"{name} must be > 0, got {getattr(self, name)}"))
        chk += [
            (self.footprint_radius_m >= 0, "footprint_radius_m must be >= 0"),
            (bool(self.eta_list), "eta_list must not be empty"),
            (all(0.0 < e <= 1.0 for e in self.eta_list), "every eta must be in (0,1]"),
            (self.k_init >= 1, f"k_init must be >= 1, got {self.k_init}"),
            (self.p >= 0, f"p must be >= 0, got {self.p}"),
            (self.i_max >= 1, f"i_max must be >= 1, got {self.i_max}"),
            (self.mc_runs >= 1, f"mc_runs must be >= 1, got {self.mc_runs}"),
            (self.alpha is None or self.alpha >= 0, f"alpha must be >= 0, got {self.alpha}"),
            (self.n_reset >= 0, f"n_reset must be >= 0, got {self.n_reset}"),
            (self.nlos_block_len >= 1 and self.beam_hold >= 1,
             "nlos_block_len and beam_hold must be >= 1"),
            (self.seed >= 0, f"seed must be >= 0, got {self.seed}"),
        ]
        n = self.pass_s * self.update_rate_Hz
        chk.append((abs(n - round(n)) <= 1e-9 and round(n) >= 1,
                    f"pass_s * update_rate_Hz must be a positive integer, got {n}"))
        for ok, msg in chk:
            if not ok:
                raise RangeError(msg)
        return self

    def with_(self, **kw) -> "ScenarioConfig":
        return replace(self, **kw)


# -- result types (harness.py:32-77) -------------------------------------------------------

@dataclass
class SnapshotRecord:
    t_s: float
    sum_rate: float
    method: str
    k_est: int
    cost_units: float


@dataclass
class TrialResult:
    method_label: str
    snapshots: list
    mean_sum_rate: float
    total_cost_units: float


@dataclass
class ComparisonRow:
    method_label: str
    eta: float | None
    savings_pct: float
    degradation_pct: float


@dataclass
class ComparisonTable:
    rows: list


@dataclass
class CampaignResult:
    labels: list
    etas: dict
    table: ComparisonTable
    pooled_rates: dict
    trial_mean_rates: dict
    mean_rate: dict
    mean_cost: dict
    mean_k_est: dict
    method_counts: dict
    decisions: dict
    n_snapshots: int
    mc_runs: int
    master_seed: int
    per_step: dict = field(default_factory=dict, repr=False)   # label -> {rates, method, k_est, cols?}


def method_label(eta: float | None) -> str:
    """harness.py:84-85."""
    return "conventional" if eta is None else f"wb_arsvd_eta{eta:g}"


def stream_seed(master_seed: int, label: str, trial_index: int) -> np.random.SeedSequence:
    """harness.py:88-92."""
    return np.random.SeedSequence(
        [int(master_seed), zlib.crc32(label.encode("utf-8")), int(trial_index)])


def ecdf(samples):
    """(value, cumulative probability) steps, duplicates collapsed onto their
    last step (harness.py:95-104).  A CUDA tensor is reduced on the device
    (sort, run-length of equal values, cumulative counts) and returned as a
    device tensor; array input keeps the host form."""
    if isinstance(samples, torch.Tensor) and samples.is_cuda:
        x = samples.reshape(-1).to(torch.float64)
        if x.numel() == 0:
            raise EmptyInputError("ecdf needs at least one sample")
        xs, _ = torch.sort(x)
        vals, cnt = torch.unique_consecutive(xs, return_counts=True)
        # elementwise IEEE division (a scalar divisor may become a reciprocal multiply)
        n = torch.full_like(vals, float(xs.numel()))
        return torch.stack([vals, torch.cumsum(cnt, 0).to(torch.float64) / n], 1)
    x = np.asarray(samples, dtype=float).ravel()
    if x.size == 0:
        raise EmptyInputError("ecdf needs at least one sample")
    xs = np.sort(x)
    vals = np.unique(xs)
    return np.column_stack([vals, np.searchsorted(xs, vals, side="right") / xs.size])


def complexity_curve(K: int) -> np.ndarray:
    """(r, cost_wb_arsvd(K, r) / K^3) for r = 1..K (harness.py:107-116)."""
    if K < 2:
        raise ValueError(f"K must be >= 2, got {K}")
    r = np.arange(1, K + 1)
    return np.column_stack([r.astype(float),
                            np.array([cost_wb_arsvd(K, int(x)) / cost_full(K) for x in r])])


# -- device pass -------------------------------------------------------------------------------

def dft_factors(n_x: int, n_y: int) -> np.ndarray:
    """The two unitary DFT matrices whose Kronecker product is the beam
    codebook (channel.py:176-190), flattened: n_x^2 then n_y^2 complex128."""
    def f(n):
        i = np.arange(n)
        return np.exp(-2j * np.pi * np.outer(i, i) / n) / math.sqrt(n)
    return np.concatenate([f(n_x).ravel(), f(n_y).ravel()])


def place_users(cfg, rng: np.random.Generator) -> np.ndarray:
    """User drop on the footprint disk (channel.py:292-311) -> [K, 5]
    (ECEF x, y, z, antenna gain dBi, Rician K linear)."""
    K = cfg.K
    radius = cfg.footprint_radius_m * np.sqrt(rng.random(K))
    bearing = 2.0 * np.pi * rng.random(K)
    lat = np.degrees((radius * np.cos(bearing)) / EARTH_RADIUS_M)
    lon = np.degrees((radius * np.sin(bearing)) / EARTH_RADIUS_M)
    out = np.empty((K, 5))
    k_lin = min(10.0 ** (float(cfg.K_R_dB) / 10.0), RICIAN_K_CAP)
    for n in range(K):
        la, lo = math.radians(float(lat[n])), math.radians(float(lon[n]))
        out[n] = (EARTH_RADIUS_M * math.cos(la) * math.cos(lo),
                  EARTH_RADIUS_M * math.cos(la) * math.sin(lo),
                  EARTH_RADIUS_M * math.sin(la), float(cfg.ut_gain_dBi), k_lin)
    return out


def leo_cfg(cfg) -> Nn.LeoCfg:
    lam = SPEED_OF_LIGHT_M_S / cfg.carrier_Hz
    R = EARTH_RADIUS_M + cfg.altitude_m
    return Nn.LeoCfg(K=cfg.K, n_x=cfg.n_x, n_y=cfg.n_y, N_RF=cfg.N_RF, beam_hold=cfg.beam_hold,
                     nlos_block=cfg.nlos_block_len, wavelength=lam,
                     spacing_m=cfg.spacing_wavelengths * lam, orbit_radius=R,
                     orbit_rate=math.sqrt(GM_EARTH / R ** 3), pass_s=cfg.pass_s,
                     dt=1.0 / cfg.update_rate_Hz,
                     min_elev_rad=math.radians(cfg.min_elevation_deg),
                     atm_loss_dB=cfg.atmospheric_loss_dB)


class DevicePass:
    """Snapshots of one pass for a set of trials, generated chunk by chunk on
    the device.  Chunks must be requested in increasing, contiguous order
    (the NLOS blocks are read sequentially from each trial's channel stream)."""

    def __init__(self, cfg, trials, master_seed: int, device):
        self.cfg, self.trials = cfg, list(trials)
        self.device = torch.device(device)
        rngs = [np.random.default_rng(stream_seed(master_seed, CHANNEL_STREAM, t))
                for t in self.trials]
        ut = np.stack([place_users(cfg, r) for r in rngs])
        self.ut = torch.from_numpy(ut).to(self.device)
        self.dft = torch.from_numpy(dft_factors(cfg.n_x, cfg.n_y)).to(self.device)
        self.lcfg = leo_cfg(cfg)
        self.nlos = DeviceOmegaStreams(rngs, self.device)
        self.next_t = 0
        self.block_normals = 2 * cfg.K * cfg.n_elements

    def generate(self, t0: int, t1: int, want_channels: bool = False) -> dict:
        if t0 != self.next_t:
            raise ValueError(f"chunks must be contiguous: expected t0={self.next_t}, got {t0}")
        nb = self.cfg.nlos_block_len
        blk0, blk1 = t0 // nb, (t1 - 1) // nb
        win = self.nlos.window((blk1 - blk0 + 1) * self.block_normals)
        out = ops.leo_snapshot(self.lcfg, len(self.trials), t0, t1 - t0, self.ut, self.dft, win,
                               want_channels)
        adv = (t1 // nb - blk0) * self.block_normals
        self.nlos.advance(torch.full((len(self.trials),), adv, dtype=torch.int64,
                                     device=self.device))
        self.next_t = t1
        return out


# -- campaign --------------------------------------------------------------------------------------

def _check_info(cfg, trials, t0, snap_info, run_infos):
    si = snap_info.cpu().numpy()
    if np.any(si == ops_info_below()):
        b, t = np.argwhere(si == ops_info_below())[0]
        raise BelowMinElevationError(f"trial {trials[b]}: UT below the elevation mask "
                                     f"{cfg.min_elevation_deg} deg at t={(t0 + t) / cfg.update_rate_Hz}")
    for inf in run_infos:
        a = inf.cpu().numpy()
        if np.any(a == 1):
            b, t = np.argwhere(a == 1)[0]
            raise SingularMatrixError(f"trial {trials[b % len(trials)]} step {t0 + t}: "
                                      "condition estimate exceeds 1e14")
        if np.any(a == 3):
            b, t = np.argwhere(a == 3)[0]
            raise ZeroPrecoderError(f"trial {trials[b % len(trials)]} step {t0 + t}: zero "
                                    "precoder norm")


def ops_info_below() -> int:
    return 5   # LRZ_INFO_BELOW_MASK


def _simulate(cfg, specs, trials, seed, device, chunk, sketch_labels=None, keep_cols=False):
    """Run every (label, eta) of ``specs`` over ``trials`` with a shared
    channel.  The WB-arSVD methods run as ONE batched runner whose rows are
    (method, trial) pairs with a per-row eta, so their in-order arSVD tails
    overlap on the GPU.  Returns label -> dict of host arrays [B, T] (rates,
    method, k_est) and stats [B, 6]."""
    dev = torch.device(device) if device is not None else torch.device("cuda", 0)
    B, T, K, R = len(trials), cfg.n_snapshots, cfg.K, cfg.N_RF
    chunk = T if chunk is None else max(1, int(chunk))
    ps = DevicePass(cfg, trials, seed, dev)
    groups = []
    conv = [(lab, eta) for lab, eta in specs if eta is None]
    wb = [(lab, eta) for lab, eta in specs if eta is not None]
    for members in (conv, wb):
        if not members:
            continue
        m = len(members)
        is_wb = members[0][1] is not None
        etas = [eta for _, eta in members for _ in trials] if is_wb else None
        # with oversampling p <= 2 the iteration count follows the sketch draw itself,
        # so speculative sketch cursors rarely survive: resolve in order from the start
        # (the energy-screen cursor walk measured slower here: 0.75 s vs 0.60 s for the
        # default campaign -- K = 16 steps are too small for its per-step latency)
        tc = TrajectoryConfig(alpha=cfg.resolved_alpha, P_t=cfg.P_t_W, eta=etas,
                              k_init=cfg.k_init, p=cfg.p, i_max=cfg.i_max, n_reset=cfg.n_reset,
                              rate_via_gram=False, delta="formula",
                              spec_passes=0 if cfg.p <= 2 else 2)
        runner = TrajectoryRunner(m * B, K, R, torch.complex128, tc, dev)
        streams = None
        if is_wb:
            gens = []
            for lab, _ in members:
                sl = (sketch_labels or {}).get(lab, lab)
                gens += [np.random.default_rng(stream_seed(seed, sl, t)) for t in trials]
            streams = DeviceOmegaStreams(gens, dev)
        groups.append(dict(labels=[lab for lab, _ in members], m=m, wb=is_wb, runner=runner,
                           streams=streams,
                           stats=torch.zeros(m * B, 6, dtype=torch.float64, device=dev),
                           noise=torch.full((m * B, K), cfg.noise_variance_W,
                                            dtype=torch.float64, device=dev),
                           rates=[], method=[], k_est=[]))
    cols = []
    rep = lambda x, m: x if m == 1 else x.repeat(m, *([1] * (x.dim() - 1)))
    main = torch.cuda.current_stream(dev)
    # the conventional group is launched first on a side stream so that its
    # batched inversions overlap the WB group's in-order arSVD on the main stream
    side = _aux_stream(dev, "side")
    for gr in groups:
        gr["stream"] = side if (not gr["wb"] and len(groups) > 1) else main
    # snapshots are generated one chunk ahead on their own stream, so chunk c+1's
    # channels, beams and NLOS draws overlap chunk c's in-order arSVD
    snap_stream = _aux_stream(dev, "snap")
    starts = list(range(0, T, chunk))

    def prefetch(t0):
        snap_stream.wait_stream(main)
        with torch.cuda.stream(snap_stream):
            sn = ps.generate(t0, min(T, t0 + chunk))
            ev = torch.cuda.Event()
            ev.record(snap_stream)
        return sn, ev

    nxt = prefetch(starts[0])
    for ci, t0 in enumerate(starts):
        t1 = min(T, t0 + chunk)
        snap, ev = nxt
        main.wait_event(ev)
        if ci + 1 < len(starts):
            nxt = prefetch(starts[ci + 1])
        infos = []
        for gr in groups:
            m, st = gr["m"], gr["stream"]
            if st is not main:
                st.wait_stream(main)
            with torch.cuda.stream(st):
                hyb = dict(H_rf=rep(snap["H_rf"], m), cols=rep(snap["cols"], m), n_x=cfg.n_x,
                           n_y=cfg.n_y, dft=ps.dft)
                H_in = rep(snap["H_eff"], m)
                if st is not main:
                    for x in (snap["H_rf"], snap["cols"], snap["H_eff"]):
                        x.record_stream(st)
                om = None
                if gr["wb"]:
                    om = gr["streams"].window((t1 - t0) * gr["runner"].normals_per_step_max())
                res = gr["runner"].run_chunk(H_in, gr["noise"], om, hybrid=hyb)
                if gr["wb"]:
                    gr["streams"].advance(res.consumed)
                ops.campaign_reduce(res.method, res.k_est, t0, K, cfg.n_reset, not gr["wb"],
                                    gr["stats"])
            gr["rates"].append(res.rates)
            gr["method"].append(res.method)
            gr["k_est"].append(res.k_est)
            infos.append(res.info)
        main.wait_stream(side)
        _check_info(cfg, trials, t0, snap["info"], infos)
        if keep_cols:
            cols.append(snap["cols"].cpu())
    out = {}
    for gr in groups:   # device tensors; the callers reduce on the device
        full = dict(rates=torch.cat(gr["rates"], 1), method=torch.cat(gr["method"], 1),
                    k_est=torch.cat(gr["k_est"], 1), stats=gr["stats"])
        for i, lab in enumerate(gr["labels"]):
            out[lab] = {k: v[i * B:(i + 1) * B] for k, v in full.items()}
    if keep_cols:
        out["_cols"] = torch.cat(cols, 1).numpy()
    return out


_STREAMS: dict = {}


def _aux_stream(dev, name: str):
    """One long-lived side stream per (device, role): the ops workspace cache is
    keyed by stream, so fresh streams per call would grow it without bound."""
    key = (dev.index if dev.index is not None else 0, name)
    if key not in _STREAMS:
        _STREAMS[key] = torch.cuda.Stream(dev)
    return _STREAMS[key]


def _dist_world():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def run_campaign(cfg, master_seed: int | None = None, workers: int = 1,
                 collect_decisions: bool = False, device=None,
                 chunk: int | None = 600) -> CampaignResult:
    """Monte-Carlo comparison of the conventional method against WB-arSVD at
    every eta of the scenario (harness.run_campaign, harness.py:313-383), on
    the GPU.  ``workers`` is accepted for signature compatibility (the
    trials run batched).  Under an initialised torch.distributed group the
    trials are sharded across ranks and gathered once at the end."""
    from .dist import gather_results, shard_trials
    del workers
    seed = cfg.seed if master_seed is None else master_seed
    etas = sorted(set(cfg.eta_list), reverse=True)
    specs = [(method_label(None), None)] + [(method_label(e), e) for e in etas]
    labels = [lab for lab, _ in specs]
    rank, world = _dist_world()
    trials = shard_trials(cfg.mc_runs, rank, world)
    if device is None and torch.cuda.is_available():
        device = torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(device) if device is not None else torch.device("cuda", 0)
    res = _simulate(cfg, specs, trials, seed, dev, chunk)
    if world > 1:
        local = {}
        for i, lab in enumerate(labels):
            for k in ("rates", "method", "k_est", "stats"):
                local[f"{i}_{k}"] = res[lab][k].cpu().numpy()
        merged = gather_results(local, trials, cfg.mc_runs, device=dev)
        res = {lab: {k: torch.from_numpy(np.ascontiguousarray(merged[f"{i}_{k}"])).to(dev)
                     for k in ("rates", "method", "k_est", "stats")}
               for i, lab in enumerate(labels)}
    # pooled means, per-trial means, mean cost / rank, counts and the comparison
    # table on the device (lrz_campaign_summary); only scalars come back
    rates_d = torch.stack([res[lab]["rates"] for lab in labels]).contiguous()
    stats_d = torch.stack([res[lab]["stats"] for lab in labels]).contiguous()
    tm_d, sm_d, tb_d = ops.campaign_summary(rates_d, stats_d)
    tm, sm, tb = tm_d.cpu().numpy(), sm_d.cpu().numpy(), tb_d.cpu().numpy()
    pooled, tmeans, mrate, mcost, mk, counts, decisions, per_step = {}, {}, {}, {}, {}, {}, {}, {}
    for i, lab in enumerate(labels):
        r = {k: v.cpu().numpy() for k, v in res[lab].items()}
        pooled[lab] = r["rates"].reshape(-1)          # the API returns the pooled samples
        tmeans[lab] = tm[i]
        mrate[lab] = float(sm[i, 0])
        mcost[lab] = float(sm[i, 1])
        mk[lab] = float(sm[i, 2])
        counts[lab] = {name: int(sm[i, 3 + j]) for j, name in enumerate(_METHOD_NAMES)}
        if collect_decisions:
            decisions[lab] = [row.astype(np.uint8) for row in r["method"]]
        per_step[lab] = r
    conv = method_label(None)
    rows = [ComparisonRow(conv, None, 0.0, 0.0)]
    for i, eta in enumerate(etas, start=1):
        rows.append(ComparisonRow(method_label(eta), eta, float(tb[i, 0]), float(tb[i, 1])))
    return CampaignResult(labels=labels, etas={method_label(e): e for e in etas} | {conv: None},
                          table=ComparisonTable(rows), pooled_rates=pooled,
                          trial_mean_rates=tmeans, mean_rate=mrate, mean_cost=mcost,
                          mean_k_est=mk, method_counts=counts, decisions=decisions,
                          n_snapshots=cfg.n_snapshots, mc_runs=cfg.mc_runs, master_seed=seed,
                          per_step=per_step)


def run_trial(cfg, eta: float | None, trial_index: int, master_seed: int | None = None,
              sketch_stream: str | None = None, device=None) -> TrialResult:
    """One pass with a single method (harness.run_trial, harness.py:259-281)."""
    seed = cfg.seed if master_seed is None else master_seed
    label = method_label(eta)
    sl = {label: sketch_stream} if sketch_stream else None
    r = _simulate(cfg, [(label, eta)], [trial_index], seed, device, None, sketch_labels=sl)[label]
    r = {k: v.cpu().numpy() for k, v in r.items()}
    T, K = cfg.n_snapshots, cfg.K
    tg = np.arange(T)
    sk = (tg > 0) & ~((cfg.n_reset > 0) & (tg % max(cfg.n_reset, 1) == 0)) if eta is not None \
        else np.zeros(T, bool)
    cost = step_costs(r["method"][0], r["k_est"][0], sk, K)
    dt = 1.0 / cfg.update_rate_Hz
    recs = [SnapshotRecord(t_s=i * dt, sum_rate=float(r["rates"][0, i]),
                           method=_METHOD_NAMES[int(r["method"][0, i])],
                           k_est=int(r["k_est"][0, i]), cost_units=float(cost[i]))
            for i in range(T)]
    return TrialResult(method_label=label, snapshots=recs,
                       mean_sum_rate=float(r["rates"][0].mean()),
                       total_cost_units=float(cost.sum()))
