"""The two condition guards decide exactly like the reference's
np.linalg.cond (lowrank.py:135-137 for the 1e14 full-inverse guard,
lowrank.py:212-216 for the 1e12 Woodbury aux guard), including cases a
hair either side of the threshold: the Frobenius bound ||X||_F ||X^-1||_F
accepts only when it proves cond_2 <= limit; otherwise cond_2 is computed by
one-sided Jacobi (csrc/linalg.cuh: cta_jacobi_cond).

Margins: 1e12 (1 +- 1e-2) for the aux; 1e14 (1 +- 1e-1) for the full inverse,
because at cond 1e14 the reference's own sigma_min (LAPACK) is only accurate to
eps * cond ~ 2 % -- a 1e-2 margin there would test rounding, not the rule."""

import numpy as np
import pytest

import paper_2512_16543_b200 as b200
from paper_2512_16543_b200 import ArSvdConfig  # noqa: F401  (API surface)
from paper_2512_16543_b200.errors import SingularAuxiliaryError, SingularMatrixError
from paper_2512_16543_b200.lowrank import GramState, LowRankFactor

pytestmark = pytest.mark.gpu


def _unitary(rng, n):
    z = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    q, r = np.linalg.qr(z)
    return q * (np.diag(r) / np.abs(np.diag(r)))


def _aux_case(rng, K, r, cond):
    """State / factor whose aux = diag(1/S) + V^H A^-1 U has 2-norm cond `cond`:
    A^-1 = I, U = V = Q (orthonormal), so aux = diag(1/S) + I; a rotation of the
    basis (Q) keeps aux diagonal in exact arithmetic but not in floating point."""
    Q = _unitary(rng, K)[:, :r]
    s_min = 1.0 / (cond * (1.0 + 1e-9) - 1.0)      # (1/s_min + 1) / (1/s_max + 1) = cond
    S = np.concatenate([[1e9], np.geomspace(1.0, 1e-3, r - 2), [s_min]])
    S = np.sort(S)[::-1].copy()
    st = GramState(A=np.eye(K, dtype=complex), A_inv=np.eye(K, dtype=complex), alpha=0.0, K=K)
    lr = LowRankFactor(U_r=Q, Sigma_r=S, V_r=Q.copy(), k_est=r)
    aux = np.diag(1.0 / S) + Q.conj().T @ Q
    return st, lr, np.linalg.cond(aux)


@pytest.mark.parametrize("rel", [-1e-2, -1e-3, 1e-3, 1e-2])
@pytest.mark.parametrize("K,r", [(16, 6), (32, 13), (64, 21)])
def test_woodbury_aux_guard_near_1e12(cuda, rel, K, r):
    rng = np.random.default_rng(K * 100 + r)
    st, lr, c_ref = _aux_case(rng, K, r, 1e12 * (1.0 + rel))
    should_raise = c_ref > 1e12
    assert (c_ref > 1e12) == (rel > 0)
    if should_raise:
        with pytest.raises(SingularAuxiliaryError):
            b200.woodbury_update(st, lr)
    else:
        out = b200.woodbury_update(st, lr)
        assert np.all(np.isfinite(out.A_inv))


@pytest.mark.parametrize("rel", [-1e-1, 1e-1])
@pytest.mark.parametrize("K", [8, 24, 48])
def test_direct_inverse_guard_near_1e14(cuda, rel, K):
    rng = np.random.default_rng(K)
    Q = _unitary(rng, K)
    lam = np.geomspace(1.0, 1.0 / (1e14 * (1.0 + rel)), K)
    A = (Q * lam) @ Q.conj().T
    A = 0.5 * (A + A.conj().T)
    c_ref = np.linalg.cond(A)
    assert (c_ref > 1e14) == (rel > 0)
    if c_ref > 1e14:
        with pytest.raises(SingularMatrixError):
            b200.direct_inverse(A)
    else:
        Ai = b200.direct_inverse(A)
        assert np.all(np.isfinite(Ai))
