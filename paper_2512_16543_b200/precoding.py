"""Drop-in for ``leorzf.precoding`` (reference pkg/src/leorzf/precoding.py).

``rzf_precoder`` and ``sum_rate`` with the reference's signatures, result
types and exceptions; F_RF = None means the fully-digital identity (SURVEY
D1), which is exactly the reference's formulas with F_RF = I.  Products run
in the sm_100a library (batched CGEMM, F-norm, SINR/rate kernels).
"""

from __future__ import annotations

from dataclasses import dataclass

import math

import numpy as np
import torch

from . import ops
from ._arrays import complex_type, device_of, is_torch, out, to_dev
from .errors import DimensionMismatchError, ZeroPrecoderError


@dataclass
class Precoder:
    """F_BB (N_RF x K) scaled so ||F_RF F_BB||_F^2 = P_t (precoding.py:18-24)."""

    F_BB: object
    scale: float
    P_t: float


@dataclass
class RateReport:
    """Per-UT Shannon rates, their sum and the SINRs (precoding.py:27-34)."""

    per_ut_rate: object
    sum_rate: float
    sinr: object


def rzf_precoder(H_eff, A_inv, F_RF, P_t: float) -> Precoder:
    """F_raw = H_eff^H A^-1, scale = sqrt(P_t) / ||F_RF F_raw||_F
    (precoding.py:37-52)."""
    K = int(H_eff.shape[0])
    if tuple(A_inv.shape) != (K, K):
        raise DimensionMismatchError(f"A_inv {tuple(A_inv.shape)} does not match K={K}")
    as_np = not is_torch(H_eff)
    ops_in = [H_eff, A_inv] + ([F_RF] if F_RF is not None else [])
    dev = device_of(*ops_in)
    ct = complex_type(*ops_in)
    H = to_dev(H_eff, ct, dev)
    F_raw = ops.cgemm(H, "H", to_dev(A_inv, ct, dev), "N")
    X = F_raw if F_RF is None else ops.cgemm(to_dev(F_RF, ct, dev), "N", F_raw, "N")
    nrm = math.sqrt(float(ops.fro2(X)[0].item()))
    if nrm == 0.0:
        raise ZeroPrecoderError("precoder has zero norm; cannot normalize power")
    scale = math.sqrt(P_t) / nrm
    return Precoder(F_BB=out(ops.axpby(scale, F_raw), as_np), scale=float(scale), P_t=float(P_t))


def sum_rate(H, F_RF, precoder: Precoder, noise) -> RateReport:
    """G = H F_RF F_BB; SINR_n = |G_nn|^2 / (sum_{i!=n} |G_ni|^2 + sigma_n^2)
    (precoding.py:55-80)."""
    K = int(H.shape[0])
    noise_np = (noise.detach().cpu().numpy() if is_torch(noise) else np.asarray(noise)).astype(float)
    if noise_np.shape != (K,):
        raise DimensionMismatchError(f"noise must have shape ({K},), got {noise_np.shape}")
    if np.any(noise_np <= 0):
        raise ValueError("noise variances must be positive")
    F_BB = precoder.F_BB
    if F_RF is not None and (F_RF.shape[0] != H.shape[1] or F_BB.shape[0] != F_RF.shape[1]):
        raise DimensionMismatchError(
            f"inconsistent shapes H {tuple(H.shape)}, F_RF {tuple(F_RF.shape)}, "
            f"F_BB {tuple(F_BB.shape)}")
    if F_RF is None and F_BB.shape[0] != H.shape[1]:
        raise DimensionMismatchError(
            f"inconsistent shapes H {tuple(H.shape)}, F_BB {tuple(F_BB.shape)}")
    as_np = not is_torch(H)
    ops_in = [H, F_BB] + ([F_RF] if F_RF is not None else [])
    dev = device_of(*ops_in)
    ct = complex_type(*ops_in)
    Hd = to_dev(H, ct, dev)
    T1 = Hd if F_RF is None else ops.cgemm(Hd, "N", to_dev(F_RF, ct, dev), "N")
    G = ops.cgemm(T1, "N", to_dev(F_BB, ct, dev), "N")
    nz = torch.from_numpy(np.ascontiguousarray(noise_np)).to(dev).reshape(1, K)
    rates, sinr, total = ops.sinr_rate(G, nz, 1)
    return RateReport(per_ut_rate=out(rates, as_np), sum_rate=float(total[0].item()),
                      sinr=out(sinr, as_np))
