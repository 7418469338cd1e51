"""Generate the golden fixtures from the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/gen_golden.py

It imports ``leorzf`` read-only from /root/reference/pkg/src (nothing is
copied into this repo) and records the reference's outputs on seeded
inputs:

* ``kat_lowrank.npz`` / ``kat_precoding.npz`` -- the instances of the
  reference's own unit tests (pkg/tests/test_lowrank.py, test_precoding.py),
  regenerated from the same seeds, with the reference's outputs;
* ``arsvd_cases.npz`` -- arsvd on assorted spectra with explicit sketch
  blocks (k_est, singular values, U S V^H, fallback flag, normals used);
* ``traj_C1.npz`` -- the C1 configuration swept with the
  reference functions under ``harness._sweep_trial`` semantics
  (harness.py:221-255), full method and WB-arSVD at several eta;
* ``traj_C2s.npz`` -- C2-shaped samples (K=32, N=256) in c128 and c64.

The GPU box never runs this script; it only reads the .npz files.
"""

from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

import leorzf  # noqa: E402  (reference, read-only)
from leorzf import lowrank as L  # noqa: E402
from leorzf import precoding as P  # noqa: E402
from leorzf import errors as E  # noqa: E402

from paper_2512_16543_b200 import scenario as S  # noqa: E402
from paper_2512_16543_b200.omega import normals_per_call_max, sketch_widths  # noqa: E402


def crandn(rng, *shape):
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / np.sqrt(2)


def random_hpd(rng, K, shift=1.0):
    B = crandn(rng, K, K)
    return B @ B.conj().T + shift * np.eye(K)


def herm_factor(rng, K, r):
    W, _ = np.linalg.qr(crandn(rng, K, r))
    s = rng.uniform(0.2, 0.9, r) * rng.choice([-1.0, 1.0], r)
    o = np.argsort(-np.abs(s))
    s, W = s[o], W[:, o]
    return W, np.abs(s), W * np.sign(s)


def h_digest(H) -> str:
    return hashlib.sha256(np.ascontiguousarray(H).tobytes()).hexdigest()


def consumed_normals(rng, snap, after, K, cfg):
    """How many normals a reference call consumed: replay candidates."""
    for n in [0] + list(np.cumsum([2 * K * d for d in
                                   sketch_widths(K, cfg.k_init, cfg.p, cfg.i_max)])):
        probe = np.random.default_rng()
        probe.bit_generator.state = snap
        if n:
            probe.standard_normal(int(n))
        if probe.bit_generator.state == after:
            return int(n)
    raise RuntimeError("could not match consumption")


def sketch_block(rng, K, cfg):
    """Worst-case normals block from a snapshot of rng (state restored)."""
    snap = rng.bit_generator.state
    block = rng.standard_normal(normals_per_call_max(K, cfg.k_init, cfg.p, cfg.i_max))
    rng.bit_generator.state = snap
    return snap, block


# ---------------------------------------------------------------------------

def gen_kat_lowrank():
    out = {}
    # direct_inverse (test_lowrank.py:48-81)
    rng = np.random.default_rng(42)
    A = random_hpd(rng, 32)
    out["di_hpd32_A"], out["di_hpd32_Ainv"] = A, L.direct_inverse(A)
    rng = np.random.default_rng(5)
    A = random_hpd(rng, 16)
    out["di_hpd16_A"], out["di_hpd16_Ainv"] = A, L.direct_inverse(A)
    rng = np.random.default_rng(9)
    Q, _ = np.linalg.qr(crandn(rng, 8, 8))
    A = (Q * np.array([3, 2, 1, 0.5, -0.5, -1, -2, -3])) @ Q.conj().T
    out["di_indef_A"], out["di_indef_Ainv"] = A, L.direct_inverse(A)
    A = np.diag([1.0, 2.0, 4.0]).astype(complex)
    out["di_diag_A"], out["di_diag_Ainv"] = A, L.direct_inverse(A)
    A = np.diag([1.0, 1e-20]).astype(complex)
    try:
        L.direct_inverse(A)
        raise AssertionError
    except E.SingularMatrixError:
        out["di_sing_A"] = A
    # gram_matrix (test_lowrank.py:84-118)
    rng = np.random.default_rng(0)
    H = crandn(rng, 8, 16)
    st = L.gram_matrix(H, 0.1)
    out["gm_H"], out["gm_A"], out["gm_Ainv"] = H, st.A, st.A_inv
    rng = np.random.default_rng(1)
    H = crandn(rng, 8, 16)
    out["gm2_H"], out["gm2_A"] = H, L.gram_matrix(H, 0.1).A
    # gram_delta (test_lowrank.py:121-153)
    rng = np.random.default_rng(4)
    H, dH = crandn(rng, 8, 16), crandn(rng, 8, 16)
    out["gd_H"], out["gd_dH"], out["gd_dA"] = H, dH, L.gram_delta(H, dH)
    rng = np.random.default_rng(6)
    H, dH = crandn(rng, 8, 16), crandn(rng, 8, 16)
    out["gd2_H"], out["gd2_dH"], out["gd2_dA"] = H, dH, L.gram_delta(H, dH)
    # woodbury (test_lowrank.py:156-221)
    rng = np.random.default_rng(7)
    A = random_hpd(rng, 16)
    U, s, V = herm_factor(rng, 16, 3)
    st = L.GramState(A=A, A_inv=np.linalg.inv(A), alpha=0.0, K=16)
    new = L.woodbury_update(st, L.LowRankFactor(U_r=U, Sigma_r=s, V_r=V, k_est=3))
    for k, v in dict(A=A, Ainv=st.A_inv, U=U, s=s, V=V, newA=new.A, newAinv=new.A_inv).items():
        out[f"wb3_{k}"] = v
    rng = np.random.default_rng(11)
    sweep = []
    for _ in range(100):
        K = int(rng.choice([4, 8, 16]))
        r = int(rng.integers(1, max(K // 2, 2)))
        A = random_hpd(rng, K)
        U, s, V = herm_factor(rng, K, r)
        st = L.GramState(A=A, A_inv=np.linalg.inv(A), alpha=0.0, K=K)
        new = L.woodbury_update(st, L.LowRankFactor(U_r=U, Sigma_r=s, V_r=V, k_est=r))
        sweep.append((K, r, A, st.A_inv, U, s, V, new.A, new.A_inv))
    out["wbs_K"] = np.array([x[0] for x in sweep])
    out["wbs_r"] = np.array([x[1] for x in sweep])
    for j, name in enumerate(["A", "Ainv", "U", "s", "V", "newA", "newAinv"]):
        flat = np.concatenate([np.ravel(x[2 + j]) for x in sweep])
        out[f"wbs_{name}"] = flat
    # update_inverse (test_lowrank.py:224-283): shared rng for data and sketch
    cases = []
    rng = np.random.default_rng(12)
    H = crandn(rng, 8, 16)
    cases.append(("zero", rng, H, np.zeros_like(H), 0.9))
    rng = np.random.default_rng(13)
    H = crandn(rng, 16, 32)
    dH = np.zeros_like(H)
    dH[0] = 0.1 * crandn(rng, 32)
    cases.append(("rank2", rng, H, dH, 0.9))
    for seed in (14, 15):
        rng = np.random.default_rng(seed)
        H = crandn(rng, 16, 16)
        Q, _ = np.linalg.qr(crandn(rng, 16, 16))
        cases.append((f"flat{seed}", rng, H, np.sqrt(16) * Q - H, 0.9))
    names = []
    for name, rng, H, dH, eta in cases:
        K = H.shape[0]
        cfg = L.ArSvdConfig(eta=eta)
        st = L.gram_matrix(H, 0.1)
        snap, block = sketch_block(rng, K, cfg)
        new, rep = L.update_inverse(st, H, dH, cfg, rng)
        used = consumed_normals(rng, snap, rng.bit_generator.state, K, cfg)
        names.append(name)
        for k, v in dict(H=H, dH=dH, omega=block, A_inv0=st.A_inv, A0=st.A,
                         newAinv=new.A_inv, newA=new.A).items():
            out[f"ui_{name}_{k}"] = v
        out[f"ui_{name}_meta"] = np.array([{"full": 0, "woodbury": 1, "none": 2}[rep.method],
                                           rep.k_est, rep.cost_units, used, eta])
    out["ui_names"] = np.array(names)
    np.savez_compressed(HERE / "kat_lowrank.npz", **out)


def gen_kat_precoding():
    out = {}
    rng = np.random.default_rng(1)
    K, N_RF, N_t = 8, 12, 64
    H = crandn(rng, K, N_RF)
    st = L.gram_matrix(H, 0.5)
    Q, _ = np.linalg.qr(crandn(rng, N_t, N_RF))
    pre = P.rzf_precoder(H, st.A_inv, Q, 3.7)
    out.update(pw_H=H, pw_Ainv=st.A_inv, pw_FRF=Q, pw_FBB=pre.F_BB, pw_scale=pre.scale)
    rng = np.random.default_rng(5)
    K, N_t, N_RF = 3, 6, 3
    H = crandn(rng, K, N_t)
    Q, _ = np.linalg.qr(crandn(rng, N_t, N_RF))
    F_BB = crandn(rng, N_RF, K)
    noise = np.array([0.5, 1.0, 2.0])
    rep = P.sum_rate(H, Q, P.Precoder(F_BB=F_BB, scale=1.0, P_t=1.0), noise)
    out.update(sr_H=H, sr_FRF=Q, sr_FBB=F_BB, sr_noise=noise, sr_rates=rep.per_ut_rate,
               sr_sinr=rep.sinr, sr_sum=rep.sum_rate)
    # fully digital (F_RF = I), random instance with many users
    rng = np.random.default_rng(77)
    K, N = 16, 64
    H = crandn(rng, K, N)
    st = L.gram_matrix(H, 1.6)
    pre = P.rzf_precoder(H, st.A_inv, np.eye(N), 1.0)
    rep = P.sum_rate(H, np.eye(N), pre, np.full(K, 0.1))
    out.update(fd_H=H, fd_Ainv=st.A_inv, fd_FBB=pre.F_BB, fd_scale=pre.scale,
               fd_rates=rep.per_ut_rate, fd_sinr=rep.sinr, fd_sum=rep.sum_rate)
    np.savez_compressed(HERE / "kat_precoding.npz", **out)


def gen_arsvd_cases():
    """arsvd on assorted spectra, with the sketch normals stored."""
    out = {}
    specs = []
    rng = np.random.default_rng(2024)
    for K, kind in [(16, "rank2"), (16, "decay"), (16, "flat"), (32, "decay"),
                    (32, "geom"), (64, "decay"), (8, "rank1"), (32, "zero")]:
        U, _ = np.linalg.qr(crandn(rng, K, K))
        if kind == "rank2":
            sv = np.r_[1.0, 0.7, np.zeros(K - 2)]
        elif kind == "rank1":
            sv = np.r_[2.0, np.zeros(K - 1)]
        elif kind == "decay":
            sv = np.exp(-0.35 * np.arange(K))
        elif kind == "geom":
            sv = 2.0 ** -np.arange(1, K + 1, dtype=float)
        elif kind == "flat":
            sv = 1.0 + 0.01 * rng.standard_normal(K)
        else:
            sv = np.zeros(K)
        sg = rng.choice([-1.0, 1.0], K)
        dA = (U * (sv * sg)) @ U.conj().T          # Hermitian, indefinite
        specs.append((K, kind, dA))
    etas = [0.999, 0.9, 0.8, 0.65]
    rows = []
    for ci, (K, kind, dA) in enumerate(specs):
        out[f"c{ci}_dA"] = dA
        for eta in etas:
            for (k_init, p, i_max) in [(2, 5, 3), (2, 1, 8), (2, 5, 4)]:
                cfg = L.ArSvdConfig(eta=eta, k_init=k_init, p=p, i_max=i_max)
                srng = np.random.default_rng([ci, int(eta * 1000), p, i_max])
                snap, block = sketch_block(srng, K, cfg)
                f = L.arsvd(dA, cfg, srng)
                used = consumed_normals(srng, snap, srng.bit_generator.state, K, cfg)
                key = f"c{ci}_e{int(eta*1000)}_p{p}_i{i_max}"
                out[key + "_omega_sha"] = np.array(h_digest(block))
                out[key + "_S"] = f.Sigma_r
                out[key + "_UVh"] = f.as_matrix() if f.k_est else np.zeros((K, K), complex)
                rows.append([ci, K, eta, k_init, p, i_max, f.k_est, int(f.used_fallback), used])
    out["rows"] = np.array(rows, dtype=float)
    np.savez_compressed(HERE / "arsvd_cases.npz", **out)


def ref_sweep(H_seq, alpha, noise, eta, sketch_rng, n_reset=1200, k_init=2, p=5, i_max=3):
    """harness._sweep_trial semantics (harness.py:221-255) with the
    reference's own functions and F_RF = I_N."""
    T, K, N = H_seq.shape
    I_N = np.eye(N)
    cfg = None if eta is None else L.ArSvdConfig(eta=eta, k_init=k_init, p=p, i_max=i_max)
    st, prev = None, None
    rates, per_ut, meth, kest, cost, used, Ainv, sinr = [], [], [], [], [], [], [], []
    for i in range(T):
        H = H_seq[i]
        if cfg is None or st is None or (n_reset > 0 and i % n_reset == 0):
            st = L.gram_matrix(H, alpha)
            m, k, c, n = "full", 0, L.cost_full(K), 0
        else:
            snap = sketch_rng.bit_generator.state
            st, rep = L.update_inverse(st, prev, H - prev, cfg, sketch_rng)
            m, k, c = rep.method, rep.k_est, rep.cost_units
            n = consumed_normals(sketch_rng, snap, sketch_rng.bit_generator.state, K, cfg)
        pre = P.rzf_precoder(H, st.A_inv, I_N, 1.0)
        rr = P.sum_rate(H, I_N, pre, noise)
        rates.append(rr.sum_rate)
        per_ut.append(rr.per_ut_rate)
        sinr.append(rr.sinr)
        meth.append({"full": 0, "woodbury": 1, "none": 2}[m])
        kest.append(k)
        cost.append(c)
        used.append(n)
        Ainv.append(st.A_inv)
        prev = H
    return dict(rates=np.array(rates), per_ut=np.array(per_ut), sinr=np.array(sinr),
                method=np.array(meth, np.uint8), k_est=np.array(kest), cost=np.array(cost),
                consumed=np.array(used), A_inv=np.array(Ainv))


def gen_traj(spec, trials, T, tag, etas, store_H, store_Ainv_for=()):
    out = {"etas": np.array([np.nan if e is None else e for e in etas]),
           "spec": np.array([spec.K, spec.N, T, spec.snr_db, spec.cap, spec.p, spec.k_init,
                             spec.i_max, spec.seed])}
    for b in trials:
        H = S.channels(spec, trials=[b], t0=0, t1=T)[0]
        out[f"t{b}_digest"] = np.array(h_digest(H))
        if store_H:
            out[f"t{b}_H"] = H
        for eta in etas:
            srng = None if eta is None else np.random.default_rng(
                S.stream_seed(spec.seed, S.method_label(eta), b))
            r = ref_sweep(H, spec.alpha, S.noise_vector(spec), eta, srng,
                          k_init=spec.k_init, p=spec.p, i_max=spec.i_max)
            lab = "full" if eta is None else f"e{int(round(eta * 1000))}"
            for k, v in r.items():
                if k == "A_inv" and eta not in store_Ainv_for:
                    continue
                out[f"t{b}_{lab}_{k}"] = v
    np.savez_compressed(HERE / f"traj_{tag}.npz", **out)


def main():
    gen_kat_lowrank()
    gen_kat_precoding()
    gen_arsvd_cases()
    gen_traj(S.C1, [0], 50, "C1", [None, 0.999, 0.9, 0.8, 0.65], store_H=True,
             store_Ainv_for=(None, 0.9, 0.65))
    c2 = S.C2
    gen_traj(c2, [0, 1], 24, "C2s", [None, 0.999, 0.9], store_H=False,
             store_Ainv_for=(0.9,))
    gen_traj(c2.with_(dtype="c64"), [0], 24, "C2s_c64", [None, 0.999, 0.9], store_H=False,
             store_Ainv_for=(None, 0.9))
    for tag in ("C2s_snr0", "C2s_snr20"):
        snr = 0.0 if tag.endswith("0") and not tag.endswith("20") else 20.0
        gen_traj(c2.with_(snr_db=snr), [0], 24, tag, [None, 0.9], store_H=False)
    print("fixtures written to", HERE)


if __name__ == "__main__":
    main()
