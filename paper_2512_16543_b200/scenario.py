"""Synthetic LEO Rician-drift channels for the BASELINE configs C1-C5.

This is the host-side channel generator the north star keeps in Python.
It follows SURVEY.md section 8(d) (no generator for these configs exists
in the reference) while reusing the reference's conventions:

* uniform planar array, element m = ix * n_y + iy centred on the origin
  (reference ``channel.py:46-59``);
* rows of H are *conjugated* array responses, so ``row @ x`` is what the
  user receives (``channel.py:9-11,128-137``) -- here with unit-modulus
  entries (no 1/sqrt(N)), so E|H_kn|^2 = beta_k;
* Rician mix sqrt(k/(1+k)) LOS + sqrt(1/(1+k)) NLOS with the NLOS energy
  matched to the LOS energy (``channel.py:140-153``);
* seeded per-trial streams keyed like ``harness.stream_seed``
  (``harness.py:88-92``): channel stream = SeedSequence([seed,
  crc32("channel"), trial]).

The NLOS scatter S is held for the whole trial by default (the analogue of
``nlos_block_len``, ``config.py:60``); ``redraw_scatter=True`` redraws it
every step (stress variant).  alpha = K / SNR, P_t = 1 and sigma_k^2 =
1 / SNR.
"""

from __future__ import annotations

import math
import zlib
from dataclasses import dataclass, field, replace

import numpy as np

CHANNEL_STREAM = "channel"


def stream_seed(master_seed: int, label: str, trial_index: int) -> np.random.SeedSequence:
    """Platform-stable seed for one (label, trial) stream; same keying as
    the reference's ``harness.stream_seed`` (harness.py:88-92)."""
    return np.random.SeedSequence(
        [int(master_seed), zlib.crc32(label.encode("utf-8")), int(trial_index)]
    )


def method_label(eta: float | None) -> str:
    """Sketch-stream label of a method (reference harness.py:84-85)."""
    return "conventional" if eta is None else f"wb_arsvd_eta{eta:g}"


@dataclass(frozen=True)
class ScenarioSpec:
    """One synthetic configuration."""

    name: str
    n_side: int                 # UPA is n_side x n_side, N = n_side**2
    K: int
    T: int
    B: int
    snr_db: float = 10.0
    kappa_db: tuple = (10.0, 10.0)          # per-user kappa ~ U[lo, hi] dB
    drift_deg: tuple = (0.05, 0.05)         # per-user drift ~ U[lo, hi] deg/step
    cone_deg: float = 20.0
    beta_span_db: float = 6.0
    tol: float = 1e-3
    cap: int = 8
    p: int = 5
    k_init: int = 2
    dtype: str = "c128"
    redraw_scatter: bool = False
    seed: int = 0

    @property
    def N(self) -> int:
        return self.n_side * self.n_side

    @property
    def alpha(self) -> float:
        return self.K / (10.0 ** (self.snr_db / 10.0))

    @property
    def noise_var(self) -> float:
        return 1.0 / (10.0 ** (self.snr_db / 10.0))

    @property
    def P_t(self) -> float:
        return 1.0

    @property
    def eta(self) -> float:
        """energy fraction eta = 1 - tol."""
        return 1.0 - self.tol

    @property
    def i_max(self) -> int:
        """cap -> i_max = 1 + log2(cap / k_init)."""
        ratio = self.cap / self.k_init
        i = int(round(math.log2(ratio)))
        if 2 ** i != ratio:
            raise ValueError(f"cap {self.cap} is not k_init * 2^j")
        return 1 + i

    def with_(self, **kw) -> "ScenarioSpec":
        return replace(self, **kw)


# The five BASELINE.json configs.
C1 = ScenarioSpec("C1", n_side=8, K=16, T=50, B=1, cap=8, dtype="c128")
C2 = ScenarioSpec("C2", n_side=16, K=32, T=200, B=64, cap=16, dtype="c128")
C3 = ScenarioSpec("C3", n_side=32, K=64, T=500, B=256, cap=16, dtype="c64",
                  kappa_db=(5.0, 15.0), drift_deg=(0.02, 0.1))
C4 = ScenarioSpec("C4", n_side=32, K=128, T=200, B=1024, cap=16, dtype="c64")
C5 = ScenarioSpec("C5", n_side=64, K=256, T=100, B=64, cap=32, dtype="c64")
CONFIGS = {s.name: s for s in (C1, C2, C3, C4, C5)}


def element_xy(n_side: int) -> np.ndarray:
    """(N, 2) element coordinates in wavelengths, lambda/2 pitch, centred,
    element m = ix * n_side + iy (channel.py:51-58 with n_x = n_y)."""
    ix, iy = np.meshgrid(np.arange(n_side), np.arange(n_side), indexing="ij")
    c = (n_side - 1) / 2.0
    return np.stack([(ix.ravel() - c) * 0.5, (iy.ravel() - c) * 0.5], axis=1)


@dataclass
class TrialDraw:
    """Per-trial random parameters (held for the whole pass)."""

    theta0: np.ndarray     # (K,) rad
    psi: np.ndarray        # (K,) rad
    phi: np.ndarray        # (K,) rad, LOS phase
    beta: np.ndarray       # (K,) linear gain
    kappa: np.ndarray      # (K,) linear Rician factor
    drift: np.ndarray      # (K,) rad / step
    rng: np.random.Generator = field(repr=False)
    scatter: np.ndarray | None = field(default=None, repr=False)  # (K, N)


def draw_trial(spec: ScenarioSpec, trial: int, scatter: bool = True) -> TrialDraw:
    """Draw one trial's user parameters from its channel stream.

    Draw order (fixed, part of the fixture contract): cos(theta0),
    psi, phi, beta_dB, kappa_dB, drift, then the scatter S (real block,
    then imaginary block, K x N row-major).  scatter=False stops before S
    (the device synthesis draws S from the same stream on the GPU)."""
    K, N = spec.K, spec.N
    rng = np.random.default_rng(stream_seed(spec.seed, CHANNEL_STREAM, trial))
    cos_lo = math.cos(math.radians(spec.cone_deg))
    theta0 = np.arccos(rng.uniform(cos_lo, 1.0, K))
    psi = rng.uniform(-math.pi, math.pi, K)
    phi = rng.uniform(-math.pi, math.pi, K)
    beta = 10.0 ** (rng.uniform(-spec.beta_span_db, 0.0, K) / 10.0)
    kappa = 10.0 ** (rng.uniform(spec.kappa_db[0], spec.kappa_db[1], K) / 10.0)
    drift = np.radians(rng.uniform(spec.drift_deg[0], spec.drift_deg[1], K))
    d = TrialDraw(theta0, psi, phi, beta, kappa, drift, rng)
    if scatter:
        d.scatter = _cn(rng, K, N)
    return d


def _cn(rng: np.random.Generator, K: int, N: int) -> np.ndarray:
    re = rng.standard_normal((K, N))
    im = rng.standard_normal((K, N))
    return math.sqrt(0.5) * (re + 1j * im)


def trial_channels(spec: ScenarioSpec, trial: int, t0: int = 0,
                   t1: int | None = None, draw: TrialDraw | None = None) -> np.ndarray:
    """Channels H_t for t in [t0, t1) of one trial: (t1-t0, K, N) complex128.

    Row k at step t is sqrt(beta_k) * ( sqrt(k/(1+k)) e^{j phi_k}
    a*(theta_k(t), psi_k) + sqrt(1/(1+k)) S_k ) with
    a*_m = exp(-j 2 pi sin(theta) (cos(psi) x_m + sin(psi) y_m))."""
    t1 = spec.T if t1 is None else t1
    d = draw if draw is not None else draw_trial(spec, trial)
    if spec.redraw_scatter and t0 != 0 and draw is None:
        raise ValueError("redraw_scatter streams must be generated from t0 = 0")
    xy = element_xy(spec.n_side)                                  # (N, 2)
    steps = np.arange(t0, t1, dtype=float)
    theta = d.theta0[None, :] + d.drift[None, :] * steps[:, None]  # (T, K)
    st = np.sin(theta)
    kx = st * np.cos(d.psi)[None, :]
    ky = st * np.sin(d.psi)[None, :]
    phase = 2.0 * math.pi * (kx[..., None] * xy[None, None, :, 0]
                             + ky[..., None] * xy[None, None, :, 1])  # (T, K, N)
    los = np.exp(-1j * phase) * np.exp(1j * d.phi)[None, :, None]
    a_los = np.sqrt(d.kappa / (1.0 + d.kappa))[None, :, None]
    a_nlos = np.sqrt(1.0 / (1.0 + d.kappa))[None, :, None]
    if spec.redraw_scatter:
        S = np.stack([d.scatter if i == 0 else _cn(d.rng, spec.K, spec.N)
                      for i in range(t1 - t0)])
    else:
        S = d.scatter[None]
    H = np.sqrt(d.beta)[None, :, None] * (a_los * los + a_nlos * S)
    return H


def channels(spec: ScenarioSpec, trials=None, t0: int = 0, t1: int | None = None) -> np.ndarray:
    """(B, T, K, N) channel tensor in the spec's dtype (c64 = a cast of the
    c128 draw, so the GPU and the oracle see identical arrays)."""
    trials = range(spec.B) if trials is None else trials
    H = np.stack([trial_channels(spec, b, t0, t1) for b in trials])
    return H.astype(np.complex64) if spec.dtype == "c64" else H


def noise_vector(spec: ScenarioSpec) -> np.ndarray:
    return np.full(spec.K, spec.noise_var)


class DeviceChannels:
    """The same channels as ``channels(spec, trials)``, synthesised on the GPU
    (``lrz_channels``): per-trial angles and gains are drawn on the host (6 K
    numbers), the scatter S from the trial's channel stream by the device RNG,
    and H_t for any step range is formed on the device -- no channel tensor
    crosses PCIe and C3/C4-sized passes can be streamed chunk by chunk."""

    def __init__(self, spec: ScenarioSpec, trials, device):
        import torch
        from . import _native as Nn
        from .omega import DeviceOmegaStreams
        if spec.redraw_scatter:
            raise NotImplementedError("device synthesis holds the scatter per trial")
        self.spec, self.trials = spec, list(trials)
        self.device = torch.device(device)
        self._torch, self._N = torch, Nn
        draws = [draw_trial(spec, t, scatter=False) for t in self.trials]
        par = np.stack([np.stack([d.theta0, d.psi, d.phi, d.beta, d.kappa, d.drift])
                        for d in draws])                                  # [B, 6, K]
        self.params = torch.from_numpy(np.ascontiguousarray(par)).to(self.device)
        st = DeviceOmegaStreams([d.rng for d in draws], self.device)
        self.scatter = st.window(2 * spec.K * spec.N)                    # [B, 2KN] (strided rows)
        if int(st._status.sum().item()):
            raise RuntimeError("device RNG could not produce the scatter window")

    def generate(self, t0: int, t1: int, out=None):
        torch = self._torch
        s = self.spec
        dt = torch.complex64 if s.dtype == "c64" else torch.complex128
        B, T = len(self.trials), t1 - t0
        H = out if out is not None else torch.empty(B, T, s.K, s.N, dtype=dt, device=self.device)
        lib = self._N.lib_for(self.device)
        self._N.check(lib.lrz_channels(0 if dt == torch.complex64 else 1, B, t0, T, s.K, s.N,
                                       s.n_side, self.params.data_ptr(), self.scatter.data_ptr(),
                                       self.scatter.stride(0), H.data_ptr(),
                                       self._N.stream_ptr(self.device)), "lrz_channels")
        return H
