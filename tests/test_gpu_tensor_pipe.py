"""The FP64 tensor-pipe (DMMA) kernels and the step-parallel Woodbury chain
against independent references on the same inputs:

* Gram H H^H + alpha I (lowrank.py:147-164) for K = 1 ... 256, complex64 and
  complex128 H, vs the complex128 product (numpy, reference op order up to
  summation): 1e-13 relative, exactly Hermitian, exactly real diagonal;
* the fused precoder + coupling + SINR kernel (precoding.py:37-80, F_RF = I)
  vs the reference formulas evaluated in complex128 (W 1e-12, rates 1e-10);
* lrz_chain_steps (step-parallel) vs lrz_chain (one CTA per trial) on the
  same plan / factors, including 'none' steps, full steps and a
  SingularAuxiliary fallback: A^-1 sequence and A state 1e-12, methods and
  info identical."""

import numpy as np
import pytest
import torch

from oracle import port
from paper_2512_16543_b200 import ops

pytestmark = pytest.mark.gpu


def crandn(rng, *shape):
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / np.sqrt(2)


def relmax(a, b):
    a, b = np.asarray(a), np.asarray(b)
    num = np.sqrt((np.abs(a - b) ** 2).sum(axis=(-1, -2)))
    den = np.sqrt((np.abs(b) ** 2).sum(axis=(-1, -2)))
    return float((num / den).max())


@pytest.mark.parametrize("K,N", [(1, 8), (7, 20), (16, 64), (32, 256), (33, 40), (64, 1024),
                                 (100, 96), (128, 512), (256, 512)])
@pytest.mark.parametrize("dtype", [np.complex64, np.complex128])
def test_gram_dmma_vs_complex128_product(cuda, K, N, dtype):
    rng = np.random.default_rng(K * 1000 + N)
    B = 5
    H = crandn(rng, B, K, N).astype(dtype)
    alpha = 0.7
    got = ops.gram(torch.from_numpy(H).to(cuda), alpha).cpu().numpy()
    Hd = H.astype(np.complex128)
    want = Hd @ Hd.conj().transpose(0, 2, 1)
    want = 0.5 * (want + want.conj().transpose(0, 2, 1)) + alpha * np.eye(K)
    assert relmax(got, want) < 1e-13
    assert np.array_equal(got, got.conj().transpose(0, 2, 1))      # exactly Hermitian
    assert np.all(np.diagonal(got, axis1=1, axis2=2).imag == 0.0)  # real diagonal


@pytest.mark.parametrize("K,N", [(4, 16), (16, 64), (32, 256), (27, 100)])
@pytest.mark.parametrize("dtype", [np.complex64, np.complex128])
def test_fused_precoder_vs_reference_formulas(cuda, K, N, dtype):
    rng = np.random.default_rng(K + N)
    B, alpha = 6, K / 10.0
    H = crandn(rng, B, K, N).astype(dtype)
    Hd = H.astype(np.complex128)
    G = Hd @ Hd.conj().transpose(0, 2, 1) + alpha * np.eye(K)
    Ainv = np.linalg.inv(G)
    noise = np.full((B, K), 0.1)
    Ht = torch.from_numpy(H).to(cuda)
    W = torch.empty(B, N, K, dtype=Ht.dtype, device=cuda)
    pr = ops.precode_rate(Ht, torch.from_numpy(Ainv).to(cuda), 1.0,
                          torch.from_numpy(noise).to(cuda), 1, W=W,
                          G_true=torch.from_numpy(G).to(cuda), alpha=alpha)
    for b in range(B):
        F_raw = Hd[b].conj().T @ Ainv[b]                     # precoding.py:47
        s = 1.0 / np.linalg.norm(F_raw, "fro")               # precoding.py:48-51
        Gc = Hd[b] @ (s * F_raw)                             # precoding.py:74
        P = np.abs(Gc) ** 2
        sig = np.diag(P)
        sinr = sig / (P.sum(axis=1) - sig + noise[b])
        rates = np.log2(1.0 + sinr)
        wtol = 1e-12 if dtype == np.complex128 else 1e-6
        assert np.linalg.norm(W[b].cpu().numpy() - F_raw) / np.linalg.norm(F_raw) < wtol
        rtol = 1e-10 if dtype == np.complex128 else 1e-6
        assert abs(pr["scale"][b].item() - s) / s < rtol
        assert np.allclose(pr["rates"][b].cpu().numpy(), rates, rtol=rtol, atol=0)
        assert np.allclose(pr["sum"][b].item(), rates.sum(), rtol=rtol, atol=0)
        assert np.allclose(pr["sinr"][b].cpu().numpy(), sinr, rtol=rtol, atol=0)


@pytest.mark.parametrize("K,N", [(40, 100), (64, 200), (100, 500), (160, 520), (256, 320)])
@pytest.mark.parametrize("dtype", [np.complex64, np.complex128])
def test_large_K_precoder_ragged_shapes(cuda, K, N, dtype):
    """K > 32: W = H^H A^-1 (3M tiled DMMA kernel at complex128, tcgen05 at
    complex64), the coupling G A^-1 (3M tiled at both dtypes), norm and rates at
    shapes that are not multiples of the 64 x 64 tile or the 16-row slab."""
    rng = np.random.default_rng(7 * K + N)
    B, alpha = 5, K / 10.0
    H = crandn(rng, B, K, N).astype(dtype)
    Hd = H.astype(np.complex128)
    G = Hd @ Hd.conj().transpose(0, 2, 1) + alpha * np.eye(K)
    Ainv = np.linalg.inv(G)
    noise = np.full((B, K), 0.1)
    Ht = torch.from_numpy(H).to(cuda)
    W = torch.empty(B, N, K, dtype=Ht.dtype, device=cuda)
    pr = ops.precode_rate(Ht, torch.from_numpy(Ainv).to(cuda), 1.0,
                          torch.from_numpy(noise).to(cuda), 1, W=W,
                          G_true=torch.from_numpy(G).to(cuda), alpha=alpha)
    wtol, rtol = (1e-12, 1e-10) if dtype == np.complex128 else (2e-5, 1e-4)
    for b in range(B):
        F_raw = Hd[b].conj().T @ Ainv[b]                     # precoding.py:47
        s = 1.0 / np.linalg.norm(F_raw, "fro")               # precoding.py:48-51
        P = np.abs(Hd[b] @ (s * F_raw)) ** 2                 # precoding.py:74
        sig = np.diag(P)
        rates = np.log2(1.0 + sig / (P.sum(axis=1) - sig + noise[b]))
        assert np.linalg.norm(W[b].cpu().numpy() - F_raw) / np.linalg.norm(F_raw) < wtol
        assert abs(pr["scale"][b].item() - s) / s < rtol
        assert np.allclose(pr["rates"][b].cpu().numpy(), rates, rtol=rtol, atol=rtol)
        assert np.allclose(pr["sum"][b].item(), rates.sum(), rtol=rtol, atol=0)


@pytest.mark.parametrize("K,D", [(48, 9), (64, 21), (128, 13)])
def test_chain_steps_equals_per_trial_chain(cuda, K, D):
    rng = np.random.default_rng(K)
    B, T = 5, 7
    H = crandn(rng, B, T, K, 3 * K)
    G = H @ H.conj().transpose(0, 1, 3, 2) + 0.5 * np.eye(K)
    A0 = G[:, 0] - 0.01 * np.eye(K)
    Ainv0 = np.linalg.inv(A0)
    # factors of a rank-r perturbation per step, descending S
    r = rng.integers(1, D + 1, size=(B, T)).astype(np.int32)
    U = np.zeros((B, T, D, K), complex)
    V = np.zeros((B, T, D, K), complex)
    S = np.zeros((B, T, D))
    for b in range(B):
        for t in range(T):
            q, _ = np.linalg.qr(crandn(rng, K, D))
            U[b, t] = q.T
            V[b, t] = q.T
            S[b, t] = np.sort(rng.uniform(0.05, 1.0, D))[::-1]
    plan = rng.choice([0, 1, 1, 1, 2], size=(B, T)).astype(np.uint8)
    plan[0, :] = 1
    # a SingularAuxiliary step: V = 0 leaves aux = diag(1/S), cond 1e14 > 1e12
    r[1, 3] = 2
    S[1, 3, :2] = [1.0, 1e-14]
    V[1, 3] = 0.0
    plan[1, 3] = 1
    Gd = torch.from_numpy(G).to(cuda)
    A_inv_full = torch.linalg.inv(Gd.reshape(-1, K, K)).reshape(B, T, K, K).contiguous()

    def run(steps):
        A_inv_seq = A_inv_full.clone(memory_format=torch.contiguous_format)  # plan 0: inv(G_t)
        A_state = torch.from_numpy(A0.copy()).to(cuda)
        method = torch.zeros(B, T, dtype=torch.uint8, device=cuda)
        info = torch.zeros(B, T, dtype=torch.int32, device=cuda)
        ops.chain(torch.from_numpy(plan).to(cuda), Gd, torch.from_numpy(Ainv0).to(cuda),
                  A_inv_seq, A_state, torch.from_numpy(U).to(cuda), torch.from_numpy(V).to(cuda),
                  torch.from_numpy(S).to(cuda), torch.from_numpy(r).to(cuda), method, info,
                  steps=steps)
        return A_inv_seq.cpu().numpy(), A_state.cpu().numpy(), method.cpu().numpy(), \
            info.cpu().numpy()

    a_seq, a_st, m_seq, i_seq = run(False)
    b_seq, b_st, m_stp, i_stp = run(True)
    assert np.array_equal(m_seq, m_stp)
    assert np.array_equal(i_seq, i_stp)
    assert m_seq[1, 3] == 0          # the SingularAuxiliary step fell back to full
    assert relmax(b_seq.reshape(-1, K, K), a_seq.reshape(-1, K, K)) < 1e-12
    assert relmax(b_st, a_st) < 1e-12
    # one Woodbury step against the oracle's woodbury_update (lowrank.py:182-227)
    b, t = 0, 0
    st = port.State(A0[b], Ainv0[b], 0.5, K)
    rr = int(r[b, t])
    lr = port.Factor(U[b, t, :rr].T.copy(), S[b, t, :rr].copy(), V[b, t, :rr].T.copy(), rr)
    want = port.woodbury_update(st, lr)
    assert np.linalg.norm(b_seq[b, t] - want.A_inv) / np.linalg.norm(want.A_inv) < 1e-10
