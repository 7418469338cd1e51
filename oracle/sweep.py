"""Per-trial time sweep with the semantics of ``harness._sweep_trial``
(reference harness.py:188-257), for the fully-digital synthetic configs.

Per step i: a full ``gram_matrix`` inversion at i = 0, on every step of the
conventional method, and every ``n_reset`` steps (harness.py:229-233);
otherwise ``update_inverse`` on dH = H_i - H_{i-1} with the *previous*
channel as H_eff (harness.py:234-241); then the precoder on H_i and the rate
on H_i (harness.py:242-243) with F_RF = I (``None``).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import port

DECISION = {"full": 0, "woodbury": 1, "none": 2}   # harness.py:29


@dataclass
class SweepRecord:
    rates: np.ndarray            # (T,)
    per_ut: np.ndarray           # (T, K)
    method: np.ndarray           # (T,) uint8 decision codes
    k_est: np.ndarray            # (T,) int
    cost: np.ndarray             # (T,)
    iters: np.ndarray            # (T,) arsvd iterations (0 = no arsvd)
    consumed: np.ndarray         # (T,) normals consumed
    fallback: np.ndarray         # (T,) bool
    margin: np.ndarray           # (T,) relative distance of the deciding cum to the target
    margin_min: np.ndarray = None  # (T,) smallest decision margin over every iteration
    A_inv: list = field(default_factory=list)
    F_BB: list = field(default_factory=list)


def _margin(f: port.Factor) -> float:
    """Smallest |cum_j - target| / target over the prefix the rank rule
    looked at -- a near-threshold tie indicator."""
    if f.s_all is None or f.e_target == 0.0:
        return np.inf
    cum = np.cumsum(f.s_all ** 2)
    return float(np.min(np.abs(cum - f.e_target)) / f.e_target)


def sweep_trial(H_seq, alpha, noise, P_t, cfg: port.Cfg | None, sketch,
                n_reset: int = 1200, keep_state: bool = False, F_RF=None) -> SweepRecord:
    """Run one method (cfg None = conventional) over one trial's channels
    H_seq (T, K, N).  ``sketch`` is that trial's Generator or FlatNormals.
    F_RF None is the identity-elided fully digital form; pass np.eye(N) for
    the reference's verbatim F_RF = I_N products."""
    T, K, _ = H_seq.shape
    rec = SweepRecord(np.zeros(T), np.zeros((T, K)), np.zeros(T, np.uint8),
                      np.zeros(T, np.int64), np.zeros(T), np.zeros(T, np.int64),
                      np.zeros(T, np.int64), np.zeros(T, bool), np.full(T, np.inf),
                      np.full(T, np.inf))
    st = None
    prev = None
    for i in range(T):
        H = H_seq[i]
        if cfg is None or st is None or (n_reset > 0 and i % n_reset == 0):
            st = port.gram_matrix(H, alpha)
            method, k, cost = "full", 0, port.cost_full(K)
        else:
            st, method, k, cost, f = port.update_inverse(st, prev, H - prev, cfg, sketch)
            rec.iters[i], rec.consumed[i] = f.iters, f.consumed
            rec.fallback[i], rec.margin[i] = f.used_fallback, _margin(f)
            rec.margin_min[i] = f.margin_min
        F_BB, _ = port.rzf_precoder(H, st.A_inv, F_RF, P_t)
        rates, total, _ = port.sum_rate(H, F_RF, F_BB, noise)
        rec.rates[i], rec.per_ut[i] = total, rates
        rec.method[i], rec.k_est[i], rec.cost[i] = DECISION[method], k, cost
        if keep_state:
            rec.A_inv.append(st.A_inv.copy())
            rec.F_BB.append(F_BB)
        prev = H
    return rec
