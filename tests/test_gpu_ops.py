"""Single-call drop-in API on the GPU vs the oracle and the reference's own
known-answer fixtures (tests/golden).  Mirrors pkg/tests/test_lowrank.py and
test_precoding.py.  Tolerances: complex128 1e-10 relative Frobenius (north
star), ranks identical."""

import numpy as np
import pytest
import torch

from conftest import load_golden, rel
from oracle import port
from paper_2512_16543_b200 import (ArSvdConfig, GramState, LowRankFactor, Precoder, arsvd,
                                   direct_inverse, gram_delta, gram_matrix, rzf_precoder,
                                   sum_rate, update_inverse, woodbury_update)
from paper_2512_16543_b200 import errors as E
from paper_2512_16543_b200.omega import normals_per_call_max

pytestmark = pytest.mark.gpu


def crandn(rng, *shape):
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / np.sqrt(2)


@pytest.fixture(scope="module")
def kl(cuda):
    return load_golden("kat_lowrank")


# -- direct_inverse (test_lowrank.py:48-81) -----------------------------------------

def test_direct_inverse_kats(kl):
    for name in ("hpd32", "hpd16", "indef", "diag"):
        got = direct_inverse(kl[f"di_{name}_A"])
        assert rel(got, kl[f"di_{name}_Ainv"]) < 1e-10, name
    assert np.allclose(direct_inverse(2.0 * np.eye(4)), 0.5 * np.eye(4))
    A = kl["di_indef_A"]
    assert np.linalg.norm(A @ direct_inverse(A) - np.eye(8)) < 1e-10
    with pytest.raises(E.SingularMatrixError):
        direct_inverse(kl["di_sing_A"])
    with pytest.raises(E.DimensionMismatchError):
        direct_inverse(np.zeros((3, 4)))


@pytest.mark.parametrize("K", [1, 7, 16, 33, 64, 65, 128, 256])
def test_direct_inverse_sizes(cuda, K):
    rng = np.random.default_rng(K)
    B = crandn(rng, K, K)
    A = B @ B.conj().T + 0.5 * np.eye(K)
    got = direct_inverse(A)
    assert rel(got, np.linalg.inv(A)) < 1e-10
    assert rel(got, port.direct_inverse(A)) < 1e-10


def test_direct_inverse_batched_torch(cuda):
    rng = np.random.default_rng(3)
    B = crandn(rng, 5, 12, 12)
    A = B @ B.conj().transpose(0, 2, 1) + np.eye(12)
    got = direct_inverse(torch.from_numpy(A).to(cuda))
    assert isinstance(got, torch.Tensor) and got.is_cuda
    assert rel(got.cpu().numpy(), np.linalg.inv(A)) < 1e-10


# -- gram_matrix / gram_delta (test_lowrank.py:84-153) --------------------------------

def test_gram_matrix_kats(kl):
    st = gram_matrix(kl["gm_H"], 0.1)
    assert rel(st.A, kl["gm_A"]) < 1e-14
    assert rel(st.A_inv, kl["gm_Ainv"]) < 1e-10
    assert st.cost_accum == 512.0
    A = gram_matrix(kl["gm2_H"], 0.1).A
    assert np.array_equal(A, A.conj().T)  # exactly Hermitian
    z = gram_matrix(np.zeros((4, 16), complex), 2.0)
    assert np.allclose(z.A, 2 * np.eye(4)) and np.allclose(z.A_inv, 0.5 * np.eye(4))
    with pytest.raises(E.SingularMatrixError):
        gram_matrix(np.zeros((4, 16), complex), 0.0)
    e = gram_matrix(np.eye(3, dtype=complex), 1.0)
    assert np.allclose(e.A_inv, 0.5 * np.eye(3))


@pytest.mark.parametrize("K,N", [(16, 64), (32, 256), (40, 100), (64, 1024), (128, 96)])
@pytest.mark.parametrize("dt", [np.complex128, np.complex64])
def test_gram_matrix_shapes(cuda, K, N, dt):
    rng = np.random.default_rng(K + N)
    H = crandn(rng, K, N).astype(dt)
    st = gram_matrix(H, 0.7)
    ref = port.gram_matrix(H, 0.7)
    tol = 1e-12 if dt == np.complex128 else 1e-5
    assert rel(st.A, ref.A) < tol
    assert rel(st.A_inv, ref.A_inv) < (1e-10 if dt == np.complex128 else 1e-4)


def test_gram_delta_kats(kl):
    for tag in ("gd", "gd2"):
        got = gram_delta(kl[f"{tag}_H"], kl[f"{tag}_dH"])
        assert rel(got, kl[f"{tag}_dA"]) < 1e-14
        assert np.array_equal(got, got.conj().T)
    rng = np.random.default_rng(2)
    H = crandn(rng, 4, 8)
    assert np.all(gram_delta(H, np.zeros_like(H)) == 0)
    dH = crandn(rng, 4, 8)
    assert np.allclose(gram_delta(np.zeros_like(dH), dH), dH @ dH.conj().T)


@pytest.mark.parametrize("K,N", [(32, 256), (64, 1024), (100, 37)])
def test_gram_delta_vs_direct_difference(cuda, K, N):
    rng = np.random.default_rng(4)
    H, dH = crandn(rng, K, N), 0.01 * crandn(rng, K, N)
    got = gram_delta(H, dH)
    Hn = H + dH
    ref = Hn @ Hn.conj().T - H @ H.conj().T
    assert rel(got, port.gram_delta(H, dH)) < 1e-12
    assert rel(got, ref) < 1e-10


# -- woodbury (test_lowrank.py:156-221) --------------------------------------------------

def test_woodbury_kats(kl):
    st = GramState(A=kl["wb3_A"], A_inv=kl["wb3_Ainv"], alpha=0.0, K=16, cost_accum=100.0)
    new = woodbury_update(st, LowRankFactor(kl["wb3_U"], kl["wb3_s"], kl["wb3_V"], 3))
    assert rel(new.A_inv, kl["wb3_newAinv"]) < 1e-10
    assert rel(new.A, kl["wb3_newA"]) < 1e-14
    assert new.cost_accum == 100.0 + 16 ** 2 + 16 ** 2 * 3 + 27 + 9 * 16


def test_woodbury_property_sweep(kl):
    """The reference's 100-instance exactness sweep (test_lowrank.py:210-221)
    against the reference outputs."""
    off = {k: 0 for k in ("A", "Ainv", "U", "s", "V", "newA", "newAinv")}
    for K, r in zip(kl["wbs_K"], kl["wbs_r"]):
        K, r = int(K), int(r)
        shp = dict(A=(K, K), Ainv=(K, K), U=(K, r), s=(r,), V=(K, r), newA=(K, K),
                   newAinv=(K, K))
        x = {}
        for k, s in shp.items():
            n = int(np.prod(s))
            x[k] = kl[f"wbs_{k}"][off[k]:off[k] + n].reshape(s)
            off[k] += n
        new = woodbury_update(GramState(x["A"], x["Ainv"], 0.0, K),
                              LowRankFactor(x["U"], x["s"].real, x["V"], r))
        assert rel(new.A_inv, x["newAinv"]) < 1e-10
        oracle = np.linalg.inv(x["A"] + (x["U"] * x["s"].real) @ x["V"].conj().T)
        assert rel(new.A_inv, oracle) < 1e-8


def test_woodbury_sherman_morrison_and_singular_aux(cuda):
    st = GramState(A=np.eye(2, dtype=complex), A_inv=np.eye(2, dtype=complex), alpha=0.0, K=2)
    e1 = np.zeros((2, 1), complex)
    e1[0, 0] = 1.0
    new = woodbury_update(st, LowRankFactor(e1, np.array([1.0]), e1.copy(), 1))
    assert np.allclose(new.A_inv, np.eye(2) - 0.5 * (e1 @ e1.conj().T))
    with pytest.raises(E.SingularAuxiliaryError):
        woodbury_update(st, LowRankFactor(e1, np.array([1.0]), -e1, 1))


# -- arsvd on assorted spectra vs the reference ------------------------------------------

def test_arsvd_cases_match_reference(cuda):
    g = load_golden("arsvd_cases")
    for row in g["rows"]:
        ci, K, eta, k_init, p, i_max, k_est, fb, used = row
        ci, K, k_init, p, i_max = int(ci), int(K), int(k_init), int(p), int(i_max)
        key = f"c{ci}_e{int(eta*1000)}_p{p}_i{i_max}"
        srng = np.random.default_rng([ci, int(eta * 1000), p, i_max])
        f = arsvd(g[f"c{ci}_dA"], ArSvdConfig(eta, k_init, p, i_max), srng)
        # the caller's generator advanced exactly as the reference's did
        probe = np.random.default_rng([ci, int(eta * 1000), p, i_max])
        probe.standard_normal(int(used))
        assert srng.bit_generator.state == probe.bit_generator.state, key
        assert f.k_est == int(k_est), (key, f.k_est, int(k_est))
        if "zero" in key or f.k_est == 0:
            continue
        assert f.used_fallback == bool(fb), key
        assert np.allclose(f.Sigma_r, g[key + "_S"], rtol=1e-10, atol=1e-13), key
        assert rel(f.as_matrix(), g[key + "_UVh"]) < 1e-9, key


def test_arsvd_flat_stream_source(cuda):
    rng = np.random.default_rng(5)
    K = 24
    Q, _ = np.linalg.qr(crandn(rng, K, K))
    dA = (Q * np.exp(-0.5 * np.arange(K))) @ Q.conj().T
    cfg = ArSvdConfig(eta=0.95, k_init=2, p=5, i_max=4)
    vals = rng.standard_normal(normals_per_call_max(K, 2, 5, 4) + 10)
    a = port.FlatNormals(vals, 3)
    b = port.FlatNormals(vals, 3)
    f = arsvd(dA, cfg, a)
    r = port.arsvd(dA, port.Cfg(0.95, 2, 5, 4), b)
    assert f.k_est == r.k_est and a.cursor == b.cursor
    assert rel(f.as_matrix(), (r.U_r * r.Sigma_r) @ r.V_r.conj().T) < 1e-10


# -- update_inverse dispatcher (test_lowrank.py:224-283) ----------------------------------

def test_update_inverse_kats(kl):
    for name in kl["ui_names"]:
        g = lambda k: kl[f"ui_{name}_{k}"]
        code, k_est, cost, used, eta = g("meta")
        st = GramState(A=g("A0"), A_inv=g("A_inv0"), alpha=0.1, K=g("H").shape[0])
        src = port.FlatNormals(g("omega"))
        new, rep = update_inverse(st, g("H"), g("dH"), ArSvdConfig(eta=eta), src)
        assert {"full": 0, "woodbury": 1, "none": 2}[rep.method] == int(code), name
        assert rep.k_est == int(k_est) and rep.cost_units == cost, name
        assert src.cursor == int(used), name
        assert rel(new.A_inv, g("newAinv")) < 1e-10, name
        if rep.method == "none":
            assert new.A_inv is st.A_inv  # aliasing, lowrank.py:347-350


# -- precoder and rate (test_precoding.py) -------------------------------------------------

def test_precoding_kats(cuda):
    g = load_golden("kat_precoding")
    pre = rzf_precoder(g["pw_H"], g["pw_Ainv"], g["pw_FRF"], 3.7)
    assert rel(pre.F_BB, g["pw_FBB"]) < 1e-12 and abs(pre.scale - float(g["pw_scale"])) < 1e-12
    assert abs(np.linalg.norm(g["pw_FRF"] @ pre.F_BB) ** 2 - 3.7) / 3.7 < 1e-8
    rep = sum_rate(g["sr_H"], g["sr_FRF"], Precoder(g["sr_FBB"], 1.0, 1.0), g["sr_noise"])
    assert np.allclose(rep.per_ut_rate, g["sr_rates"], rtol=0, atol=1e-12)
    assert abs(rep.sum_rate - float(g["sr_sum"])) < 1e-12
    pre = rzf_precoder(g["fd_H"], g["fd_Ainv"], None, 1.0)
    assert rel(pre.F_BB, g["fd_FBB"]) < 1e-12
    rep = sum_rate(g["fd_H"], None, pre, np.full(16, 0.1))
    assert abs(rep.sum_rate - float(g["fd_sum"])) < 1e-10 * abs(rep.sum_rate)
    assert np.allclose(rep.sinr, g["fd_sinr"], rtol=1e-9)


def test_precoding_edge_cases(cuda):
    with pytest.raises(E.ZeroPrecoderError):
        rzf_precoder(np.zeros((2, 4), complex), np.eye(2, dtype=complex),
                     np.zeros((8, 4), complex), 1.0)
    rep = sum_rate(np.array([[1.0 + 0j]]), np.array([[1.0 + 0j]]),
                   Precoder(np.array([[1.0 + 0j]]), 1.0, 1.0), np.array([1.0]))
    assert abs(rep.sum_rate - 1.0) < 1e-12
    H = np.zeros((2, 4), complex)
    F = np.zeros((4, 2), complex)
    pre = Precoder(np.zeros((2, 2), complex), 1.0, 1.0)
    with pytest.raises(E.DimensionMismatchError):
        sum_rate(H, F, pre, np.array([1.0]))
    with pytest.raises(ValueError):
        sum_rate(H, F, pre, np.array([1.0, 0.0]))
