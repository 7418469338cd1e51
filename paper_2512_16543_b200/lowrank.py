"""Drop-in for ``leorzf.lowrank`` (reference pkg/src/leorzf/lowrank.py).

Same names, signatures, dataclasses, cost model and exceptions; the
arithmetic runs in the sm_100a library (K1 Gram, K1' Gram correction,
K2+K3 arSVD, K4 Woodbury, K5 Hermitian inverse).  numpy in -> numpy out,
torch CUDA in -> torch CUDA out.  Additions over the reference:
``gram_matrix`` / ``direct_inverse`` / ``gram_delta`` accept leading batch
dimensions, and ``arsvd`` / ``update_inverse`` accept any object with
``values`` / ``cursor`` (a flat pre-drawn normal stream) in
place of the Generator.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import ops
from ._arrays import complex_type, device_of, is_torch, np_dtype, out, to_dev
from .errors import (DimensionMismatchError, SingularAuxiliaryError, SingularMatrixError,
                     INFO_SINGULAR, INFO_SINGULAR_AUX)
from .omega import GeneratorBudget, normals_per_call_max

COND_LIMIT_FULL = 1e14     # lowrank.py:27
COND_LIMIT_AUX = 1e12      # lowrank.py:28


@dataclass
class GramState:
    """A = H H^H + alpha I, its maintained inverse, alpha, K and the cost
    counter (lowrank.py:31-44)."""

    A: object
    A_inv: object
    alpha: float
    K: int
    cost_accum: float = 0.0


@dataclass
class LowRankFactor:
    """U_r diag(Sigma_r) V_r^H with rank k_est (lowrank.py:47-67)."""

    U_r: object
    Sigma_r: object
    V_r: object
    k_est: int
    used_fallback: bool = False

    @classmethod
    def empty(cls, K: int) -> "LowRankFactor":
        z = np.zeros((K, 0), dtype=complex)
        return cls(U_r=z, Sigma_r=np.zeros(0), V_r=z.copy(), k_est=0)

    def as_matrix(self):
        """Dense U diag(S) V^H (testing use)."""
        if is_torch(self.U_r):
            return (self.U_r * self.Sigma_r) @ self.V_r.conj().transpose(-1, -2)
        return (self.U_r * self.Sigma_r) @ self.V_r.conj().T


@dataclass
class ArSvdConfig:
    """eta in (0, 1], k_init >= 1, p >= 0, i_max >= 1 (lowrank.py:70-88)."""

    eta: float
    k_init: int = 2
    p: int = 1
    i_max: int = 8

    def __post_init__(self):
        if not 0.0 < self.eta <= 1.0:
            raise ValueError(f"eta must be in (0,1], got {self.eta}")
        if self.k_init < 1:
            raise ValueError(f"k_init must be >= 1, got {self.k_init}")
        if self.p < 0:
            raise ValueError(f"p must be >= 0, got {self.p}")
        if self.i_max < 1:
            raise ValueError(f"i_max must be >= 1, got {self.i_max}")


@dataclass
class UpdateReport:
    """Path taken ('woodbury' | 'full' | 'none'), rank and cost (lowrank.py:91-98)."""

    method: str
    k_est: int
    cost_units: float


def cost_full(K: int) -> float:
    """K^3 (lowrank.py:101-103)."""
    return float(K) ** 3


def cost_wb_arsvd(K: int, r: int) -> float:
    """K^2 + K^2 r + r^3 + r^2 K (lowrank.py:106-110)."""
    K, r = float(K), float(r)
    return K ** 2 + K ** 2 * r + r ** 3 + r ** 2 * K


def sketch_cost(K: int, r: int) -> float:
    """K^2 r + r^2 K (lowrank.py:113-118)."""
    K, r = float(K), float(r)
    return K ** 2 * r + r ** 2 * K


def _require_square(A) -> int:
    shp = tuple(A.shape)
    if len(shp) < 2 or shp[-1] != shp[-2]:
        raise DimensionMismatchError(f"expected a square matrix, got {shp}")
    return shp[-1]


def _raise_singular(info: torch.Tensor, what: str) -> None:
    bad = (info == INFO_SINGULAR)
    if bool(bad.any()):
        idx = torch.nonzero(bad.reshape(-1))[0].item()
        raise SingularMatrixError(
            f"{what}: condition estimate exceeds {COND_LIMIT_FULL:.1e} (item {idx})")


def direct_inverse(A):
    """Hermitian inverse with the 1e14 condition guard (lowrank.py:127-144)."""
    K = _require_square(A)
    as_np = not is_torch(A)
    dev = device_of(A)
    Ainv, info = ops.herm_inverse(to_dev(A, np.complex128, dev), COND_LIMIT_FULL)
    _raise_singular(info, "direct_inverse")
    return out(Ainv, as_np, np_dtype(A))


def gram_matrix(H_eff, alpha: float) -> GramState:
    """A = H H^H (symmetrised) + alpha I and its inverse (lowrank.py:147-164)."""
    if len(tuple(H_eff.shape)) < 2:
        raise DimensionMismatchError(f"H_eff must be 2-D, got {tuple(H_eff.shape)}")
    if alpha < 0:
        raise ValueError(f"alpha must be >= 0, got {alpha}")
    K = int(H_eff.shape[-2])
    as_np = not is_torch(H_eff)
    dev = device_of(H_eff)
    H = to_dev(H_eff, complex_type(H_eff), dev)
    A = ops.gram(H, alpha)
    Ainv, info = ops.herm_inverse(A, COND_LIMIT_FULL)
    # alpha = 0 with rank-deficient H has cond = inf >> 1e14 (lowrank.py:158-159)
    _raise_singular(info, "gram_matrix")
    return GramState(A=out(A, as_np), A_inv=out(Ainv, as_np), alpha=float(alpha), K=K,
                     cost_accum=cost_full(K))


def gram_delta(H_eff, dH_eff):
    """H dH^H + dH H^H + dH dH^H (lowrank.py:167-179); result dtype follows
    numpy promotion of the inputs."""
    if tuple(H_eff.shape) != tuple(dH_eff.shape):
        raise DimensionMismatchError(
            f"shape mismatch: H_eff {tuple(H_eff.shape)} vs dH_eff {tuple(dH_eff.shape)}")
    as_np = not is_torch(H_eff)
    dev = device_of(H_eff, dH_eff)
    ct = complex_type(H_eff, dH_eff)
    Hd, dHd = to_dev(H_eff, ct, dev), to_dev(dH_eff, ct, dev)
    lead = tuple(Hd.shape[:-2])
    K, Nn = Hd.shape[-2:]
    dA = ops.gram_delta(Hd.reshape(-1, K, Nn), dHd.reshape(-1, K, Nn), 0).reshape(*lead, K, K)
    res_dt = np.result_type(np_dtype(H_eff), np_dtype(dH_eff))
    return out(dA, as_np, res_dt)


def _sketch_block(rng, n_max: int):
    """Worst-case normal block + a commit callback (Generator or flat stream)."""
    if isinstance(rng, np.random.Generator):
        bud = GeneratorBudget(rng, n_max)
        return bud.block, bud.commit
    if hasattr(rng, "values") and hasattr(rng, "cursor"):
        vals = np.asarray(rng.values, dtype=np.float64)
        c = int(rng.cursor)
        blk = vals[c:c + n_max]
        if blk.size < n_max:
            blk = np.concatenate([blk, np.full(n_max - blk.size, np.nan)])

        def commit(used, rng=rng, avail=vals.size - c):
            if used > avail:
                raise IndexError("omega stream exhausted")
            rng.cursor = int(rng.cursor) + int(used)

        return blk, commit
    raise TypeError("rng must be a numpy Generator or a flat normal stream (values, cursor)")


def _arsvd_device(dA_dev: torch.Tensor, cfg: ArSvdConfig, rng):
    K = dA_dev.shape[-1]
    n_max = normals_per_call_max(K, cfg.k_init, cfg.p, cfg.i_max)
    block, commit = _sketch_block(rng, n_max)
    dev = dA_dev.device
    omega = torch.from_numpy(np.ascontiguousarray(block)).to(dev).reshape(1, -1)
    cursor = torch.zeros(1, dtype=torch.int64, device=dev)
    res = ops.arsvd(dA_dev.reshape(1, K, K).contiguous(), omega, cursor, cfg.eta, cfg.k_init,
                    cfg.p, cfg.i_max)
    k = int(res["k_est"][0].item())
    commit(int(res["consumed"][0].item()))
    return res, k


def _factor_from(res, k: int, K: int, as_np: bool) -> LowRankFactor:
    if k == 0:
        f = LowRankFactor.empty(K)
        if not as_np:
            dev = res["U"].device
            f = LowRankFactor(torch.zeros(K, 0, dtype=torch.complex128, device=dev),
                              torch.zeros(0, dtype=torch.float64, device=dev),
                              torch.zeros(K, 0, dtype=torch.complex128, device=dev), 0)
        return f
    U = res["U"][0, :k].transpose(0, 1).contiguous()
    V = res["V"][0, :k].transpose(0, 1).contiguous()
    S = res["S"][0, :k].contiguous()
    return LowRankFactor(U_r=out(U, as_np), Sigma_r=out(S, as_np), V_r=out(V, as_np), k_est=k,
                         used_fallback=bool(res["fallback"][0].item()))


def arsvd(dA, cfg: ArSvdConfig, rng) -> LowRankFactor:
    """Adaptive randomised SVD (lowrank.py:243-316); consumes exactly the
    normals the reference would from ``rng``."""
    K = _require_square(dA)
    if len(tuple(dA.shape)) != 2:
        raise DimensionMismatchError("arsvd takes one K x K matrix")
    as_np = not is_torch(dA)
    dev = device_of(dA)
    res, k = _arsvd_device(to_dev(dA, np.complex128, dev), cfg, rng)
    return _factor_from(res, k, K, as_np)


def _woodbury_device(A, Ainv, U, V, S, r):
    """U, V: (K, r) device tensors -> column-major [1][r][K] layout."""
    Uc = U.transpose(0, 1).contiguous().unsqueeze(0)
    Vc = V.transpose(0, 1).contiguous().unsqueeze(0)
    Sd = S.to(torch.float64).reshape(1, r).contiguous()
    rr = torch.tensor([r], dtype=torch.int32, device=Ainv.device)
    A_out, Ai_out, info = ops.woodbury(A.unsqueeze(0) if A is not None else None,
                                       Ainv.unsqueeze(0), Uc, Vc, Sd, rr)
    return (A_out[0] if A_out is not None else None), Ai_out[0], int(info[0].item())


def woodbury_update(state: GramState, lr: LowRankFactor) -> GramState:
    """(A + U S V^H)^-1 by the Woodbury identity (lowrank.py:182-227)."""
    r = int(lr.k_est)
    if r < 1:
        raise ValueError("woodbury_update requires a factor of rank >= 1")
    K = state.K
    if (tuple(lr.U_r.shape) != (K, r) or tuple(lr.V_r.shape) != (K, r)
            or tuple(lr.Sigma_r.shape) != (r,)):
        raise DimensionMismatchError(
            f"factor shapes {tuple(lr.U_r.shape)}/{tuple(lr.Sigma_r.shape)}/"
            f"{tuple(lr.V_r.shape)} inconsistent with K={K}, r={r}")
    as_np = not is_torch(state.A_inv)
    dev = device_of(state.A_inv, lr.U_r)
    c = np.complex128
    A_out, Ai_out, info = _woodbury_device(
        to_dev(state.A, c, dev), to_dev(state.A_inv, c, dev), to_dev(lr.U_r, c, dev),
        to_dev(lr.V_r, c, dev), to_dev(lr.Sigma_r, np.float64, dev), r)
    if info == INFO_SINGULAR_AUX:
        raise SingularAuxiliaryError(
            f"auxiliary condition estimate exceeds {COND_LIMIT_AUX:.1e}")
    return GramState(A=out(A_out, as_np), A_inv=out(Ai_out, as_np), alpha=state.alpha, K=K,
                     cost_accum=state.cost_accum + cost_wb_arsvd(K, r))


def update_inverse(state: GramState, H_eff, dH_eff, cfg: ArSvdConfig, rng):
    """Alg. 2 dispatcher (lowrank.py:319-373)."""
    K = state.K
    if int(H_eff.shape[0]) != K:
        raise DimensionMismatchError(f"H_eff has {H_eff.shape[0]} rows, state expects K={K}")
    if tuple(H_eff.shape) != tuple(dH_eff.shape):
        raise DimensionMismatchError(
            f"shape mismatch: H_eff {tuple(H_eff.shape)} vs dH_eff {tuple(dH_eff.shape)}")
    as_np = not is_torch(state.A_inv)
    dev = device_of(state.A_inv, H_eff, dH_eff)
    ct = complex_type(H_eff, dH_eff)
    H = to_dev(H_eff, ct, dev)
    dH = to_dev(dH_eff, ct, dev)
    dA = ops.gram_delta(H, dH, 0)[0]
    res, k = _arsvd_device(dA, cfg, rng)
    if k == 0:
        cost = cost_wb_arsvd(K, 0)
        return (GramState(A=state.A, A_inv=state.A_inv, alpha=state.alpha, K=K,
                          cost_accum=state.cost_accum + cost),
                UpdateReport(method="none", k_est=0, cost_units=cost))
    if k / K <= 0.5:
        c = np.complex128
        U = res["U"][0, :k].transpose(0, 1)
        V = res["V"][0, :k].transpose(0, 1)
        A_out, Ai_out, info = _woodbury_device(to_dev(state.A, c, dev),
                                               to_dev(state.A_inv, c, dev), U, V,
                                               res["S"][0, :k], k)
        if info != INFO_SINGULAR_AUX:
            cost = cost_wb_arsvd(K, k)
            return (GramState(A=out(A_out, as_np), A_inv=out(Ai_out, as_np), alpha=state.alpha,
                              K=K, cost_accum=state.cost_accum + cost),
                    UpdateReport(method="woodbury", k_est=k, cost_units=cost))
    # full branch: Gram of H_eff + dH_eff (lowrank.py:361-373)
    H_new = ops.axpby(1.0, H, 1.0, dH)
    A_new = ops.gram(H_new, state.alpha)
    Ainv, info = ops.herm_inverse(A_new, COND_LIMIT_FULL)
    _raise_singular(info, "update_inverse")
    cost = cost_full(K) + sketch_cost(K, k)
    return (GramState(A=out(A_new, as_np), A_inv=out(Ainv, as_np), alpha=state.alpha, K=K,
                      cost_accum=state.cost_accum + cost),
            UpdateReport(method="full", k_est=k, cost_units=cost))
