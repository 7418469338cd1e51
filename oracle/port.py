"""numpy/scipy restatement of leorzf's L1 numerical core (test oracle).

Every routine names the reference lines it follows.  Numerics use the same
LAPACK entry points as the reference (zgesdd for cond/svd, zpotrf/zpotrs,
zgeqrf, zgesv, zgemm) so that, on the same inputs, results agree with the
reference to rounding -- this is checked against fixtures generated from
the reference itself (tests/golden/).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.linalg as sla

COND_LIMIT_FULL = 1e14     # lowrank.py:27
COND_LIMIT_AUX = 1e12      # lowrank.py:28
SQRT_HALF = float(np.sqrt(0.5))


class OracleSingular(Exception):
    """SingularMatrixError analogue (lowrank.py:136-137,158-159)."""


class OracleSingularAux(Exception):
    """SingularAuxiliaryError analogue (lowrank.py:213-216)."""


class OracleZeroPrecoder(Exception):
    """ZeroPrecoderError analogue (precoding.py:49-50)."""


class OracleShape(Exception):
    """DimensionMismatchError analogue."""


@dataclass
class State:
    """GramState (lowrank.py:31-44)."""
    A: np.ndarray
    A_inv: np.ndarray
    alpha: float
    K: int
    cost_accum: float = 0.0


@dataclass
class Factor:
    """LowRankFactor (lowrank.py:47-67) plus the sketch bookkeeping the
    device path reports (iterations run, normals consumed)."""
    U_r: np.ndarray
    Sigma_r: np.ndarray
    V_r: np.ndarray
    k_est: int
    used_fallback: bool = False
    iters: int = 0
    consumed: int = 0
    s_all: np.ndarray | None = None        # full singular values of the last sketch
    e_target: float = 0.0
    # smallest relative distance of any decision quantity to its threshold over
    # every iteration run (cumsum(s^2) vs the energy target, and on the
    # fallback tail s vs s_0 K eps): the near-tie indicator of SURVEY A.1
    margin_min: float = np.inf


@dataclass
class Cfg:
    """ArSvdConfig (lowrank.py:70-88)."""
    eta: float
    k_init: int = 2
    p: int = 1
    i_max: int = 8


# -- cost model (lowrank.py:101-118) ------------------------------------------

def cost_full(K):
    return float(K) ** 3


def cost_wb_arsvd(K, r):
    K, r = float(K), float(r)
    return K * K + K * K * r + r ** 3 + r * r * K


def sketch_cost(K, r):
    K, r = float(K), float(r)
    return K * K * r + r * r * K


# -- sketch sources ------------------------------------------------------------

class FlatNormals:
    """A flat normal stream with a cursor; ``standard_normal(shape)`` reads
    the next prod(shape) values row-major, exactly like a Generator would
    have produced them (chunking invariance)."""

    def __init__(self, values: np.ndarray, cursor: int = 0):
        self.values = np.asarray(values, dtype=np.float64)
        self.cursor = int(cursor)

    def standard_normal(self, shape):
        n = int(np.prod(shape))
        if self.cursor + n > self.values.size:
            raise IndexError("omega stream exhausted")
        out = self.values[self.cursor:self.cursor + n].reshape(shape)
        self.cursor += n
        return out


# -- inversion (lowrank.py:121-164) -------------------------------------------

def direct_inverse(A):
    """cond via SVD, then Cholesky solve against I, else Hermitian solve
    (lowrank.py:127-144)."""
    if A.ndim != 2 or A.shape[0] != A.shape[1]:
        raise OracleShape(A.shape)
    cond = np.linalg.cond(A)
    if not np.isfinite(cond) or cond > COND_LIMIT_FULL:
        raise OracleSingular(cond)
    ident = np.eye(A.shape[0], dtype=A.dtype)
    try:
        fac = sla.cho_factor(A, check_finite=False)
        return sla.cho_solve(fac, ident, check_finite=False)
    except sla.LinAlgError:
        return sla.solve(A, ident, assume_a="her", check_finite=False)


def hermitian_gram(H, alpha):
    """H H^H symmetrised plus alpha I (lowrank.py:160-162 / 365-366).
    The alpha I term is complex128, so a c64 H promotes the result."""
    K = H.shape[0]
    G = H @ H.conj().T
    G = 0.5 * (G + G.conj().T)
    return G + alpha * np.eye(K, dtype=complex)


def gram_matrix(H, alpha):
    """lowrank.py:147-164."""
    if H.ndim != 2:
        raise OracleShape(H.shape)
    if alpha < 0:
        raise ValueError("alpha must be >= 0")
    K = H.shape[0]
    if alpha == 0.0 and np.linalg.matrix_rank(H) < K:
        raise OracleSingular("rank")
    A = hermitian_gram(H, alpha)
    return State(A=A, A_inv=direct_inverse(A), alpha=float(alpha), K=K,
                 cost_accum=cost_full(K))


def gram_delta(H, dH):
    """H dH^H + (H dH^H)^H + dH dH^H (lowrank.py:167-179)."""
    if H.shape != dH.shape:
        raise OracleShape((H.shape, dH.shape))
    c = H @ dH.conj().T
    return c + c.conj().T + dH @ dH.conj().T


# -- Woodbury (lowrank.py:182-227) --------------------------------------------

def woodbury_update(st: State, f: Factor) -> State:
    r = f.k_est
    if r < 1:
        raise ValueError("rank >= 1 required")
    K = st.K
    if f.U_r.shape != (K, r) or f.V_r.shape != (K, r) or f.Sigma_r.shape != (r,):
        raise OracleShape("factor")
    Ai = st.A_inv
    AiU = Ai @ f.U_r
    aux = np.diag(1.0 / f.Sigma_r).astype(complex)
    aux += f.V_r.conj().T @ AiU
    c = np.linalg.cond(aux)
    if not np.isfinite(c) or c > COND_LIMIT_AUX:
        raise OracleSingularAux(c)
    aux_inv = np.linalg.inv(aux)
    VhAi = f.V_r.conj().T @ Ai
    return State(A=st.A + (f.U_r * f.Sigma_r) @ f.V_r.conj().T,
                 A_inv=Ai - (AiU @ aux_inv) @ VhAi,
                 alpha=st.alpha, K=K,
                 cost_accum=st.cost_accum + cost_wb_arsvd(K, r))


# -- adaptive randomized SVD (lowrank.py:230-316) -------------------------------

def orthonormal_basis(Y):
    """Reduced QR with the R diagonal rotated real non-negative
    (lowrank.py:230-240)."""
    Q, R = np.linalg.qr(Y)
    dg = np.diagonal(R)
    mag = np.abs(dg)
    ph = np.where(mag > 0, dg / np.where(mag > 0, mag, 1.0), 1.0)
    return Q * ph


def arsvd(dA, cfg: Cfg, rng) -> Factor:
    """Algorithm 1 of the paper as implemented at
    lowrank.py:243-316.  ``rng`` is a numpy Generator or a FlatNormals."""
    if dA.ndim != 2 or dA.shape[0] != dA.shape[1]:
        raise OracleShape(dA.shape)
    K = dA.shape[0]
    energy = np.linalg.norm(dA, "fro") ** 2
    if energy == 0.0:
        z = np.zeros((K, 0), dtype=complex)
        return Factor(z, np.zeros(0), z.copy(), 0)
    target = cfg.eta * energy
    k0, used = cfg.k_init, 0
    s = Uap = Vh = None
    mmin = np.inf
    for it in range(cfg.i_max):
        d = min(k0 + cfg.p, K)
        om = SQRT_HALF * (rng.standard_normal((K, d)) + 1j * rng.standard_normal((K, d)))
        used += 2 * K * d
        Q = orthonormal_basis(dA @ om)
        Uh, s, Vh = np.linalg.svd(Q.conj().T @ dA, full_matrices=False)
        Uap = Q @ Uh
        cum = np.cumsum(s ** 2)
        mmin = min(mmin, float(np.min(np.abs(cum - target)) / target))
        hit = np.flatnonzero(cum >= target)
        if hit.size:
            r = int(hit[0]) + 1
            return Factor(Uap[:, :r], s[:r].copy(), Vh[:r].conj().T, r, False,
                          it + 1, used, s.copy(), float(target), mmin)
        k0 *= 2
    floor = s[0] * K * np.finfo(float).eps
    r = max(int(np.count_nonzero(s > floor)), 1)
    if floor > 0:
        mmin = min(mmin, float(np.min(np.abs(s - floor)) / floor))
    return Factor(Uap[:, :r], s[:r].copy(), Vh[:r].conj().T, r, True,
                  cfg.i_max, used, s.copy(), float(target), mmin)


# -- dispatcher (lowrank.py:319-373) ----------------------------------------------

def update_inverse(st: State, H, dH, cfg: Cfg, rng):
    """Alg. 2.  Returns (state, method, k_est, cost, factor)."""
    K = st.K
    if H.shape[0] != K:
        raise OracleShape(H.shape)
    f = arsvd(gram_delta(H, dH), cfg, rng)
    if f.k_est == 0:
        c = cost_wb_arsvd(K, 0)
        return (State(st.A, st.A_inv, st.alpha, K, st.cost_accum + c), "none", 0, c, f)
    if f.k_est / K <= 0.5:
        try:
            new = woodbury_update(st, f)
            return new, "woodbury", f.k_est, cost_wb_arsvd(K, f.k_est), f
        except OracleSingularAux:
            pass
    A = hermitian_gram(H + dH, st.alpha)
    c = cost_full(K) + sketch_cost(K, f.k_est)
    return (State(A, direct_inverse(A), st.alpha, K, st.cost_accum + c), "full",
            f.k_est, c, f)


# -- precoder and rate (precoding.py:37-80) ----------------------------------------

def rzf_precoder(H_eff, A_inv, F_RF, P_t):
    """F_raw = H^H A^-1 scaled to ||F_RF F_raw||_F^2 = P_t.  F_RF=None is the
    fully-digital identity.  Returns (F_BB, scale)."""
    K = H_eff.shape[0]
    if A_inv.shape != (K, K):
        raise OracleShape(A_inv.shape)
    F_raw = H_eff.conj().T @ A_inv
    nrm = np.linalg.norm(F_raw if F_RF is None else F_RF @ F_raw, "fro")
    if nrm == 0.0:
        raise OracleZeroPrecoder()
    scale = np.sqrt(P_t) / nrm
    return scale * F_raw, float(scale)


def sum_rate(H, F_RF, F_BB, noise):
    """SINR_n = |G_nn|^2 / (sum_{i!=n} |G_ni|^2 + sigma_n^2), G = H F_RF F_BB
    (precoding.py:55-80).  Returns (per_ut_rate, sum, sinr)."""
    K = H.shape[0]
    noise = np.asarray(noise, dtype=float)
    if noise.shape != (K,):
        raise OracleShape(noise.shape)
    if np.any(noise <= 0):
        raise ValueError("noise variances must be positive")
    G = H @ F_BB if F_RF is None else H @ F_RF @ F_BB
    pw = np.abs(G) ** 2
    sig = np.diagonal(pw)
    sinr = sig / (pw.sum(axis=1) - sig + noise)
    rates = np.log2(1.0 + sinr)
    return rates, float(rates.sum()), sinr
