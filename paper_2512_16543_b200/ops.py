"""Device-tensor operators: one function per C-ABI entry point.

Inputs are torch CUDA tensors (contiguous, batch-major); outputs are new
CUDA tensors.  Everything is stream-ordered on the current torch stream and
never synchronises the host.  The drop-in API (lowrank.py / precoding.py)
and the batched trajectory runner (trajectory.py) are built on these.
"""

from __future__ import annotations

import os

import ctypes as C
import math

import torch

from . import _native as N

_WS: dict = {}

# Kernel launches issued through this module (bench.py reports it as
# gpu_launches): incremented by the number of kernels each entry point launches.
LAUNCHES = [0]


def dmma_active() -> bool:
    """The K <= 32 Gram / precoder kernels run on the FP64 tensor pipe (both
    dtypes) unless LRZ_SIMT_FP64=1 selects the SIMT kernels (A/B runs)."""
    return os.environ.get("LRZ_SIMT_FP64") != "1"


def _count(n: int = 1) -> None:
    LAUNCHES[0] += n


def workspace(device, nbytes: int, slot: str = "main") -> torch.Tensor:
    """Grow-only per-(device, slot) scratch buffer."""
    # per stream: runners on different streams must not share scratch
    key = (device.index if device.index is not None else 0,
           torch.cuda.current_stream(device).cuda_stream, slot)
    buf = _WS.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)
        _WS[key] = buf
    return buf


def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.complex64:
        return N.C64
    if t.dtype == torch.complex128:
        return N.C128
    raise TypeError(f"expected complex64/complex128, got {t.dtype}")


def _chk(t: torch.Tensor, name: str) -> torch.Tensor:
    if not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t


def _items(t: torch.Tensor, name: str) -> tuple[int, int]:
    """(count, element stride) of a [B, r, c] batch whose matrices are
    contiguous but whose batch stride may be larger (views like x[:, 0])."""
    if not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dim() != 3 or t.stride(2) != 1 or t.stride(1) != t.shape[2]:
        raise ValueError(f"{name} must be [B, r, c] with contiguous matrices")
    if t.shape[0] > 1 and t.stride(0) < t.shape[1] * t.shape[2]:
        raise ValueError(f"{name}: overlapping batch stride")
    return t.shape[0], (t.stride(0) if t.shape[0] > 1 else t.shape[1] * t.shape[2])


def _batch(t: torch.Tensor, tail: int):
    lead = t.shape[:-tail]
    return lead, int(math.prod(lead)) if lead else 1


def d_max_for(K: int, k_init: int, p: int, i_max: int) -> int:
    """Widest sketch the schedule can reach (lowrank.py:283,302)."""
    return min(k_init * 2 ** (i_max - 1) + p, K)


def gram(H: torch.Tensor, alpha: float, out: torch.Tensor | None = None) -> torch.Tensor:
    """K1: H H^H + alpha I (complex128 out) over leading batch dims."""
    _chk(H, "H")
    lead, B = _batch(H, 2)
    K, Nn = H.shape[-2:]
    A = out if out is not None else torch.empty(*lead, K, K, dtype=torch.complex128,
                                                 device=H.device)
    lib = N.lib_for(H.device)
    N.check(lib.lrz_gram(_dt(H), B, K, Nn, H.data_ptr(), K * Nn, float(alpha), A.data_ptr(),
                         K * K, N.stream_ptr(H.device)), "lrz_gram")
    _count(1)  # K <= 32: warp per item; K > 32: warp per lower 32 x 32 block
    return A


def gram_delta(P: torch.Tensor, Q: torch.Tensor, mode: int,
               out: torch.Tensor | None = None) -> torch.Tensor:
    """K1': Gram correction, complex128 out.  mode 0: (H, dH); mode 1: (H_prev, H_cur).
    P, Q, out: [B, ., .] batches (matrices contiguous, batch stride free)."""
    if P.dim() == 2:
        P, Q = P.unsqueeze(0), Q.unsqueeze(0)
        if out is not None:
            out = out.unsqueeze(0)
    if P.shape != Q.shape or P.dtype != Q.dtype:
        raise ValueError("P/Q shape or dtype mismatch")
    B, ps = _items(P, "P")
    _, qs = _items(Q, "Q")
    K, Nn = P.shape[-2:]
    dA = out if out is not None else torch.empty(B, K, K, dtype=torch.complex128,
                                                  device=P.device)
    _, as_ = _items(dA, "out")
    lib = N.lib_for(P.device)
    N.check(lib.lrz_gram_delta(_dt(P), B, K, Nn, P.data_ptr(), ps, Q.data_ptr(), qs,
                               mode, dA.data_ptr(), as_, N.stream_ptr(P.device)),
            "lrz_gram_delta")
    _count(1)
    return dA


def herm_inverse(A: torch.Tensor, cond_limit: float = 1e14, mask: torch.Tensor | None = None,
                 out: torch.Tensor | None = None, info: torch.Tensor | None = None):
    """K5: batched Hermitian inverse with the cond guard; returns (A_inv, info)."""
    _chk(A, "A")
    if A.dtype != torch.complex128:
        raise TypeError("herm_inverse works on complex128")
    lead, B = _batch(A, 2)
    K = A.shape[-1]
    if out is None:
        out = torch.empty_like(A)
    if info is None:
        info = torch.zeros(lead if lead else (1,), dtype=torch.int32, device=A.device)
    lib = N.lib_for(A.device)
    ws = workspace(A.device, lib.lrz_workspace_bytes(N.WS_INVERSE, N.C128, B, K, 0, 0), "inv")
    N.check(lib.lrz_herm_inverse(B, K, A.data_ptr(), K * K, out.data_ptr(), K * K,
                                 info.data_ptr(), float(cond_limit), N.ptr(mask), ws.data_ptr(),
                                 N.stream_ptr(A.device)), "lrz_herm_inverse")
    # warp (K <= 32) or cluster (64 < K <= 256) fast path + the CTA kernel for flagged items
    _count(2 if (K <= 32 or 64 < K <= 256) else 1)
    return out, info


def _arsvd_cfg(eta, k_init: int, p: int, i_max: int, D: int, omega_len: int = 0):
    """ArsvdCfg for a scalar eta, or per omega row (a float64 CUDA tensor);
    omega_len > 0 bounds the normals a call may read per omega row."""
    if isinstance(eta, torch.Tensor):
        if not eta.is_cuda or eta.dtype != torch.float64 or not eta.is_contiguous():
            raise ValueError("per-row eta must be a contiguous float64 CUDA tensor")
        return N.ArsvdCfg(1.0, int(k_init), int(p), int(i_max), int(D), eta.data_ptr(),
                          int(omega_len))
    return N.ArsvdCfg(float(eta), int(k_init), int(p), int(i_max), int(D), None, int(omega_len))


def arsvd(dA: torch.Tensor, omega: torch.Tensor, cursor: torch.Tensor, eta, k_init: int,
          p: int, i_max: int, omega_row: torch.Tensor | None = None,
          mask: torch.Tensor | None = None, out: dict | None = None,
          want_factor: bool | int = True, hermitian: bool = False) -> dict:
    """K2+K3 over a flat batch of items.  dA [B,K,K] c128; omega [R,L] f64;
    cursor [B] int64; omega_row [B] int32 (row of omega per item, default = item).
    want_factor 2: screen-only cursor-resolution mode (iters / consumed estimates)."""
    _chk(dA, "dA")
    if not omega.is_cuda or omega.dim() != 2 or omega.stride(1) != 1:
        raise ValueError("omega must be a [R, L] CUDA tensor with contiguous rows")
    B = dA.shape[0]
    K = dA.shape[-1]
    D = d_max_for(K, k_init, p, i_max)
    dev = dA.device
    if out is None:
        out = dict(
            U=torch.empty(B, D, K, dtype=torch.complex128, device=dev),
            V=torch.empty(B, D, K, dtype=torch.complex128, device=dev),
            S=torch.zeros(B, D, dtype=torch.float64, device=dev),
            k_est=torch.zeros(B, dtype=torch.int32, device=dev),
            iters=torch.zeros(B, dtype=torch.int32, device=dev),
            fallback=torch.zeros(B, dtype=torch.int32, device=dev),
            consumed=torch.zeros(B, dtype=torch.int64, device=dev),
        )
    cfg = _arsvd_cfg(eta, k_init, p, i_max, D, omega.shape[1])
    lib = N.lib_for(dev)
    nbytes = lib.lrz_workspace_bytes(N.WS_ARSVD, N.C128, B, K, 0, D)
    ws = workspace(dev, nbytes, "arsvd")
    N.check(lib.lrz_arsvd(B, K, dA.data_ptr(), K * K, omega.data_ptr(), omega.stride(0),
                          N.ptr(omega_row), cursor.data_ptr(), C.byref(cfg), out["U"].data_ptr(),
                          out["V"].data_ptr(), out["S"].data_ptr(), out["k_est"].data_ptr(),
                          out["iters"].data_ptr(), out["fallback"].data_ptr(),
                          out["consumed"].data_ptr(), N.ptr(mask), int(want_factor),
                          int(hermitian), ws.data_ptr(), N.stream_ptr(dev)), "lrz_arsvd")
    # screening front end (sketch GEMM [+ W GEMM for K > 32] + screen) + the exact kernel
    front = hermitian and int(want_factor) != 1 and D <= 40
    # K <= 32: fused sketch + screen + exact; K > 32: Omega gather + Y + W GEMMs on
    # DMMA (SIMT: sketch + W GEMM) + screen + exact; want_factor 2: no exact kernel
    _count(((3 if K <= 32 else (5 if dmma_active() else 4)) if front else 1)
           - (1 if int(want_factor) == 2 else 0))
    out["D"] = D
    return out


def arsvd_seq(dA: torch.Tensor, omega: torch.Tensor, is_sketch: torch.Tensor,
              first_unverified: torch.Tensor, cursor: torch.Tensor, iters_pred: torch.Tensor,
              eta, k_init: int, p: int, i_max: int, out: dict,
              want_factor: bool = False) -> dict:
    """In-order arSVD of each trial's unverified suffix.  dA [B,T,K,K] c128
    contiguous; omega [B,L] (contiguous rows); is_sketch [B,T] u8;
    first_unverified [B] i32; cursor [B,T] i64 and iters_pred [B,T] i32 (in/out);
    out: the flat [B*T] result dict of ``arsvd``."""
    _chk(dA, "dA")
    if not omega.is_cuda or omega.dim() != 2 or omega.stride(1) != 1:
        raise ValueError("omega must be a [B, L] CUDA tensor with contiguous rows")
    B, T, K = dA.shape[0], dA.shape[1], dA.shape[-1]
    D = d_max_for(K, k_init, p, i_max)
    dev = dA.device
    cfg = _arsvd_cfg(eta, k_init, p, i_max, D, omega.shape[1])
    lib = N.lib_for(dev)
    ws = workspace(dev, lib.lrz_workspace_bytes(N.WS_ARSVD, N.C128, B * T, K, 0, D), "arsvd")
    N.check(lib.lrz_arsvd_seq(B, T, K, dA.data_ptr(), omega.data_ptr(), omega.stride(0),
                              C.byref(cfg), _chk(is_sketch, "is_sketch").data_ptr(),
                              _chk(first_unverified, "first_unverified").data_ptr(),
                              _chk(cursor, "cursor").data_ptr(),
                              _chk(iters_pred, "iters_pred").data_ptr(), out["U"].data_ptr(),
                              out["V"].data_ptr(), out["S"].data_ptr(), out["k_est"].data_ptr(),
                              out["iters"].data_ptr(), out["fallback"].data_ptr(),
                              out["consumed"].data_ptr(), int(want_factor), ws.data_ptr(),
                              N.stream_ptr(dev)), "lrz_arsvd_seq")
    _count(1)
    return out


def arsvd_walk(dA: torch.Tensor, omega: torch.Tensor, is_sketch: torch.Tensor,
               first_unverified: torch.Tensor, cursor: torch.Tensor, iters_pred: torch.Tensor,
               eta, k_init: int, p: int, i_max: int) -> None:
    """Cursor walk (K <= 32): cursors and iteration counts of each trial's steps
    from first_unverified on, in order, from the CholeskyQR energy screen alone.
    dA [B,T,K,K]; omega [B,L]; cursor [B,T] i64 and iters_pred [B,T] i32 (in/out)."""
    _chk(dA, "dA")
    B, T, K = dA.shape[0], dA.shape[1], dA.shape[-1]
    D = d_max_for(K, k_init, p, i_max)
    cfg = _arsvd_cfg(eta, k_init, p, i_max, D, omega.shape[1])
    lib = N.lib_for(dA.device)
    N.check(lib.lrz_arsvd_walk(B, T, K, dA.data_ptr(), omega.data_ptr(), omega.stride(0),
                               C.byref(cfg), _chk(is_sketch, "is_sketch").data_ptr(),
                               _chk(first_unverified, "first_unverified").data_ptr(),
                               _chk(cursor, "cursor").data_ptr(),
                               _chk(iters_pred, "iters_pred").data_ptr(),
                               N.stream_ptr(dA.device)), "lrz_arsvd_walk")
    _count(1)


def walk_ok(K: int, k_init: int, p: int, i_max: int) -> bool:
    """lrz_arsvd_walk's limits: K <= 32, every sketch width <= 24."""
    if K > 32:
        return False
    k0 = k_init
    for _ in range(i_max):
        if min(k0 + p, K) > 24:
            return False
        k0 *= 2
    return True


def woodbury(A: torch.Tensor | None, A_inv: torch.Tensor, U: torch.Tensor, V: torch.Tensor,
             S: torch.Tensor, r: torch.Tensor):
    """K4 over a batch: returns (A_out or None, A_inv_out, info)."""
    B, K = A_inv.shape[0], A_inv.shape[-1]
    D = U.shape[1]
    dev = A_inv.device
    A_inv_out = torch.empty_like(A_inv)
    A_out = torch.empty_like(A) if A is not None else None
    info = torch.zeros(B, dtype=torch.int32, device=dev)
    lib = N.lib_for(dev)
    ws = workspace(dev, lib.lrz_workspace_bytes(N.WS_WOODBURY, N.C128, B, K, 0, D), "wb")
    N.check(lib.lrz_woodbury(B, K, D, N.ptr(A), A_inv.data_ptr(), K * K, U.data_ptr(),
                             V.data_ptr(), S.data_ptr(), r.data_ptr(), N.ptr(A_out),
                             A_inv_out.data_ptr(), info.data_ptr(), ws.data_ptr(),
                             N.stream_ptr(dev)), "lrz_woodbury")
    _count(1)
    return A_out, A_inv_out, info


def chain(plan, G, A_inv_prev, A_inv_seq, A_state, U, V, S, r, method, info,
          steps: bool = False):
    """Sequential Woodbury chain over [B, T] steps (in place): one CTA per trial,
    or with ``steps`` the step-parallel form (products batched over trials)."""
    for t_, n_ in ((plan, "plan"), (G, "G"), (A_inv_prev, "A_inv_prev"), (A_inv_seq, "A_inv_seq"),
                   (U, "U"), (V, "V"), (S, "S"), (r, "r"), (method, "method"), (info, "info")):
        _chk(t_, n_)
    if A_state is not None:
        _chk(A_state, "A_state")
    B, T = plan.shape
    K = A_inv_seq.shape[-1]
    D = U.shape[-2]
    dev = plan.device
    lib = N.lib_for(dev)
    ws = workspace(dev, lib.lrz_workspace_bytes(N.WS_CHAIN, N.C128, B, K, 0, D), "chain")
    fn = lib.lrz_chain_steps if steps else lib.lrz_chain
    N.check(fn(B, T, K, D, plan.data_ptr(), G.data_ptr(), A_inv_prev.data_ptr(),
               A_inv_seq.data_ptr(), N.ptr(A_state), U.data_ptr(), V.data_ptr(),
               S.data_ptr(), r.data_ptr(), method.data_ptr(), info.data_ptr(),
               ws.data_ptr(), N.stream_ptr(dev)), "lrz_chain")
    # step-parallel: 2 GEMMs + core + apply + fallback per step
    _count(5 * T if steps else 1)


def precode_rate(H: torch.Tensor, A_inv: torch.Tensor, P_t: float, noise: torch.Tensor,
                 noise_div: int, W: torch.Tensor | None = None, want_sinr: bool = True,
                 G_true: torch.Tensor | None = None, alpha: float = 0.0):
    """K6 over a flat batch: H [B,K,N], A_inv [B,K,K] c128, noise [R,K] f64 with
    row = item // noise_div.  Returns dict(W (unscaled F_raw or None), scale,
    rates [B,K], sinr, sum [B], info)."""
    _chk(H, "H")
    _chk(A_inv, "A_inv")
    _chk(noise, "noise")
    if G_true is not None:
        _chk(G_true, "G_true")
    if W is not None:
        _chk(W, "W")
    B, K, Nn = H.shape
    dev = H.device
    lib = N.lib_for(dev)
    scale = torch.empty(B, dtype=torch.float64, device=dev)
    rates = torch.empty(B, K, dtype=torch.float64, device=dev)
    sinr = torch.empty(B, K, dtype=torch.float64, device=dev) if want_sinr else None
    total = torch.empty(B, dtype=torch.float64, device=dev)
    info = torch.zeros(B, dtype=torch.int32, device=dev)
    ws = workspace(dev, lib.lrz_workspace_bytes(N.WS_PRECODE, _dt(H), B, K, Nn, 0), "precode")
    N.check(lib.lrz_precode_rate(_dt(H), B, K, Nn, H.data_ptr(), K * Nn, A_inv.data_ptr(), K * K,
                                 float(P_t), noise.data_ptr(), int(noise_div), N.ptr(W), Nn * K,
                                 N.ptr(G_true), float(alpha),
                                 scale.data_ptr(), rates.data_ptr(), N.ptr(sinr),
                                 total.data_ptr(), info.data_ptr(), ws.data_ptr(),
                                 N.stream_ptr(dev)), "lrz_precode_rate")
    # complex128, K <= 32 with the Gram shortcut: one fused DMMA kernel (dmma.cu)
    fused = G_true is not None and K <= 32 and dmma_active()
    _count(1 if fused else 3)
    return dict(W=W, scale=scale, rates=rates, sinr=sinr, sum=total, info=info)


_OP = {"N": 0, "T": 1, "H": 2}


def cgemm(A: torch.Tensor, opA: str, Bm: torch.Tensor, opB: str) -> torch.Tensor:
    """Batched C = op(A) op(B) over leading dims (same dtype)."""
    _chk(A, "A")
    _chk(Bm, "B")
    if A.dtype != Bm.dtype:
        raise TypeError("cgemm operands must share a dtype")
    lead, nb = _batch(A, 2)
    ar, ac = A.shape[-2:]
    br, bc = Bm.shape[-2:]
    M, Ka = (ar, ac) if opA == "N" else (ac, ar)
    Kb, Nn = (br, bc) if opB == "N" else (bc, br)
    if Ka != Kb:
        raise ValueError("inner dimensions differ")
    Cm = torch.empty(*lead, M, Nn, dtype=A.dtype, device=A.device)
    sB = 0 if Bm.dim() == 2 and nb > 1 else br * bc
    lib = N.lib_for(A.device)
    N.check(lib.lrz_cgemm(_dt(A), nb, M, Nn, Ka, _OP[opA], A.data_ptr(), ac, ar * ac, _OP[opB],
                          Bm.data_ptr(), bc, sB, Cm.data_ptr(), Nn, M * Nn,
                          N.stream_ptr(A.device)), "lrz_cgemm")
    _count(1)
    return Cm


def axpby(a: float, X: torch.Tensor, b: float = 0.0, Y: torch.Tensor | None = None,
          out: torch.Tensor | None = None):
    """Z = a X + b Y elementwise (contiguous operands of one dtype)."""
    _chk(X, "X")
    if Y is not None:
        _chk(Y, "Y")
    Z = out if out is not None else torch.empty_like(X)
    _chk(Z, "out")
    lib = N.lib_for(X.device)
    N.check(lib.lrz_axpby(_dt(X), X.numel(), float(a), X.data_ptr(), float(b), N.ptr(Y),
                          Z.data_ptr(), N.stream_ptr(X.device)), "lrz_axpby")
    _count(1)
    return Z


def fro2(X: torch.Tensor, tail: int = 2) -> torch.Tensor:
    _chk(X, "X")
    lead, nb = _batch(X, tail)
    n = int(math.prod(X.shape[-tail:]))
    out = torch.empty(lead if lead else (1,), dtype=torch.float64, device=X.device)
    lib = N.lib_for(X.device)
    N.check(lib.lrz_fro2(_dt(X), nb, n, X.data_ptr(), n, out.data_ptr(),
                         N.stream_ptr(X.device)), "lrz_fro2")
    _count(1)
    return out


def sinr_rate(G: torch.Tensor, noise: torch.Tensor, noise_div: int,
              scale: torch.Tensor | None = None):
    _chk(G, "G")
    lead, nb = _batch(G, 2)
    K = G.shape[-1]
    dev = G.device
    rates = torch.empty(*lead, K, dtype=torch.float64, device=dev)
    sinr = torch.empty(*lead, K, dtype=torch.float64, device=dev)
    total = torch.empty(lead if lead else (1,), dtype=torch.float64, device=dev)
    lib = N.lib_for(dev)
    N.check(lib.lrz_sinr_rate(_dt(G), nb, K, G.data_ptr(), K * K, N.ptr(scale), noise.data_ptr(),
                              int(noise_div), rates.data_ptr(), sinr.data_ptr(),
                              total.data_ptr(), N.stream_ptr(dev)), "lrz_sinr_rate")
    _count(1)
    return rates, sinr, total


def plan(is_sketch: torch.Tensor, k_est: torch.Tensor, K: int, out: torch.Tensor | None = None):
    """Dispatcher decision per step (lowrank.py:345-359) as a uint8 plan."""
    pl = out if out is not None else torch.empty_like(is_sketch)
    lib = N.lib_for(is_sketch.device)
    N.check(lib.lrz_plan(is_sketch.numel(), K, is_sketch.data_ptr(), k_est.data_ptr(),
                         pl.data_ptr(), N.stream_ptr(is_sketch.device)), "lrz_plan")
    _count(1)
    return pl


SPEC_VOTE_W = 16   # LRZ_SPEC_VOTE_W


def spec_verify(is_sketch, iters_pred, iters_act, cursor, cursor0, first_unverified, active,
                pending, K, eta, k_init, p, i_max, votes=None):
    """votes: optional uint8 [B, T, SPEC_VOTE_W] tally (majority re-prediction)."""
    B, T = is_sketch.shape
    dev = is_sketch.device
    cfg = _arsvd_cfg(eta, k_init, p, i_max, d_max_for(K, k_init, p, i_max))
    lib = N.lib_for(dev)
    if votes is not None:
        _chk(votes, "votes")
        assert votes.shape == (B, T, SPEC_VOTE_W) and votes.dtype == torch.uint8
    N.check(lib.lrz_spec_verify_vote(B, T, K, C.byref(cfg), is_sketch.data_ptr(),
                                     iters_pred.data_ptr(), N.ptr(iters_act), cursor.data_ptr(),
                                     cursor0.data_ptr(), first_unverified.data_ptr(),
                                     active.data_ptr(), pending.data_ptr(), N.ptr(votes),
                                     N.stream_ptr(dev)),
            "lrz_spec_verify")
    _count(1)


# -- hybrid LEO pass (leo.cu) ------------------------------------------------------------

def leo_snapshot(cfg, B: int, t0: int, T: int, ut: torch.Tensor, dft: torch.Tensor,
                 nlos: torch.Tensor, want_channels: bool = False):
    """Snapshots of steps [t0, t0+T) for B trials.  cfg: _native.LeoCfg; ut
    [B,K,5] f64; dft: c128 [nx*nx + ny*ny]; nlos [B, L] f64 (row stride free)
    starting at NLOS block t0 // nlos_block.  Returns dict(H_eff, H_rf
    [B,T,K,N_RF] c128, cols [B,T,N_RF] int32, info [B,T] int32, and H,
    H_tilde [B,T,K,N] when want_channels)."""
    dev = ut.device
    K, R, Nn = cfg.K, cfg.N_RF, cfg.n_x * cfg.n_y
    if nlos.stride(-1) != 1:
        raise ValueError("nlos rows must be contiguous")
    c128 = torch.complex128
    out = dict(H_eff=torch.empty(B, T, K, R, dtype=c128, device=dev),
               H_rf=torch.empty(B, T, K, R, dtype=c128, device=dev),
               cols=torch.empty(B, T, R, dtype=torch.int32, device=dev),
               info=torch.zeros(B, T, dtype=torch.int32, device=dev))
    if want_channels:
        out["H"] = torch.empty(B, T, K, Nn, dtype=c128, device=dev)
        out["H_tilde"] = torch.empty(B, T, K, Nn, dtype=c128, device=dev)
    lib = N.lib_for(dev)
    N.check(lib.lrz_leo_snapshot(cfg, B, t0, T, ut.data_ptr(), dft.data_ptr(), nlos.data_ptr(),
                                 nlos.stride(0), out["H_eff"].data_ptr(), out["H_rf"].data_ptr(),
                                 out["cols"].data_ptr(), out["info"].data_ptr(),
                                 N.ptr(out.get("H")), N.ptr(out.get("H_tilde")),
                                 N.stream_ptr(dev)), "lrz_leo_snapshot")
    _count(1)
    return out


def hybrid_precode_rate(H_eff: torch.Tensor, A_inv: torch.Tensor, H_rf: torch.Tensor,
                        cols: torch.Tensor, n_x: int, n_y: int, dft: torch.Tensor, P_t: float,
                        noise: torch.Tensor, noise_div: int, want_F: bool = False):
    """Flat batch: H_eff / H_rf [B,K,R] c128, A_inv [B,K,K] c128, cols [B,R]
    int32.  Returns dict(F_BB [B,R,K] or None, scale, rates [B,K], sum [B], info)."""
    for t, nm in ((H_eff, "H_eff"), (A_inv, "A_inv"), (H_rf, "H_rf"), (cols, "cols")):
        _chk(t, nm)
    B, K, R = H_eff.shape
    dev = H_eff.device
    F = torch.empty(B, R, K, dtype=torch.complex128, device=dev) if want_F else None
    scale = torch.empty(B, dtype=torch.float64, device=dev)
    rates = torch.empty(B, K, dtype=torch.float64, device=dev)
    total = torch.empty(B, dtype=torch.float64, device=dev)
    info = torch.zeros(B, dtype=torch.int32, device=dev)
    lib = N.lib_for(dev)
    N.check(lib.lrz_hybrid_precode_rate(B, K, R, n_x, n_y, H_eff.data_ptr(), A_inv.data_ptr(),
                                        H_rf.data_ptr(), cols.data_ptr(), dft.data_ptr(),
                                        float(P_t), noise.data_ptr(), int(noise_div), N.ptr(F),
                                        scale.data_ptr(), rates.data_ptr(), total.data_ptr(),
                                        info.data_ptr(), N.stream_ptr(dev)),
            "lrz_hybrid_precode_rate")
    _count(1)
    return dict(F_BB=F, scale=scale, rates=rates, sum=total, info=info)


def campaign_reduce(method: torch.Tensor, k_est: torch.Tensor, t_base: int, K: int,
                    n_reset: int, conventional: bool, stats: torch.Tensor) -> torch.Tensor:
    """Accumulate per-trial (cost, k_sum, k_count, n_full, n_woodbury, n_none)
    of a [B,T] chunk into stats [B,6] f64."""
    B, T = method.shape
    lib = N.lib_for(method.device)
    N.check(lib.lrz_campaign_reduce(B, T, int(t_base), K, int(n_reset), int(bool(conventional)),
                                    _chk(method, "method").data_ptr(),
                                    _chk(k_est, "k_est").data_ptr(), stats.data_ptr(),
                                    N.stream_ptr(method.device)), "lrz_campaign_reduce")
    _count(1)
    return stats


# -- per-kernel event timing (lrz_prof_*) ------------------------------------------------

def prof_enable(on: bool = True, device=None) -> None:
    """Bracket every instrumented launch with CUDA events on its stream."""
    lib = N.lib_for(device if device is not None else torch.device("cuda", 0))
    lib.lrz_prof_enable(1 if on else 0)


def prof_collect(device=None) -> dict:
    """{kernel: (total ms, launches)} of the launches since prof_enable."""
    lib = N.lib_for(device if device is not None else torch.device("cuda", 0))
    out = {}
    raw = lib.lrz_prof_collect()
    for part in (raw.decode() if raw else "").split(";"):
        if "=" not in part:
            continue
        name, v = part.split("=", 1)
        ms, n = v.split(":")
        out[name] = (float(ms), int(n))
    return out


# -- fused entry points (fused.cu) ---------------------------------------------------------

def update_inverse_fused(H: torch.Tensor, dH: torch.Tensor, alpha: float, A: torch.Tensor,
                         A_inv: torch.Tensor, omega: torch.Tensor, cursor: torch.Tensor, eta,
                         k_init: int, p: int, i_max: int) -> dict:
    """lrz_update_inverse over a flat batch: H, dH [B,K,N]; A, A_inv [B,K,K] c128;
    omega [B,L] f64 (row b = item b's stream); cursor [B] i64."""
    for t_, n_ in ((H, "H"), (dH, "dH"), (A, "A"), (A_inv, "A_inv"), (cursor, "cursor")):
        _chk(t_, n_)
    if not omega.is_cuda or omega.dim() != 2 or omega.stride(1) != 1:
        raise ValueError("omega must be a [B, L] CUDA tensor with contiguous rows")
    B, K, Nn = H.shape
    dev = H.device
    D = d_max_for(K, k_init, p, i_max)
    cfg = _arsvd_cfg(eta, k_init, p, i_max, D, omega.shape[1])
    lib = N.lib_for(dev)
    out = dict(A=torch.empty_like(A), A_inv=torch.empty_like(A_inv),
               method=torch.empty(B, dtype=torch.uint8, device=dev),
               k_est=torch.empty(B, dtype=torch.int32, device=dev),
               consumed=torch.empty(B, dtype=torch.int64, device=dev),
               cost=torch.empty(B, dtype=torch.float64, device=dev),
               info=torch.empty(B, dtype=torch.int32, device=dev))
    ws = workspace(dev, lib.lrz_update_inverse_ws(_dt(H), B, K, Nn, D), "fused_ui")
    N.check(lib.lrz_update_inverse(_dt(H), B, K, Nn, H.data_ptr(), dH.data_ptr(), float(alpha),
                                   A.data_ptr(), A_inv.data_ptr(), omega.data_ptr(),
                                   omega.stride(0), cursor.data_ptr(), C.byref(cfg),
                                   out["A"].data_ptr(), out["A_inv"].data_ptr(),
                                   out["method"].data_ptr(), out["k_est"].data_ptr(),
                                   out["consumed"].data_ptr(), out["cost"].data_ptr(),
                                   out["info"].data_ptr(), ws.data_ptr(), N.stream_ptr(dev)),
            "lrz_update_inverse")
    _count(8)
    return out


def trajectory_chunk(H: torch.Tensor, alpha: float, P_t: float, noise: torch.Tensor, t0: int,
                     n_reset: int, eta, k_init: int, p: int, i_max: int,
                     omega: torch.Tensor | None, A_inv_state: torch.Tensor,
                     A_state: torch.Tensor | None, G_prev: torch.Tensor | None,
                     keep_A_inv: bool = False) -> dict:
    """lrz_trajectory: one chunk H [B,T,K,N] of the in-order sweep (eta None =
    conventional).  A_inv_state / A_state are updated in place; returns the
    per-step outputs and G_last for the next chunk."""
    _chk(H, "H")
    _chk(noise, "noise")
    _chk(A_inv_state, "A_inv_state")
    B, T, K, Nn = H.shape
    dev = H.device
    D = 1 if eta is None else d_max_for(K, k_init, p, i_max)
    cfg = None if eta is None else _arsvd_cfg(eta, k_init, p, i_max, D, omega.shape[1])
    lib = N.lib_for(dev)
    out = dict(rates=torch.empty(B, T, dtype=torch.float64, device=dev),
               per_ut=torch.empty(B, T, K, dtype=torch.float64, device=dev),
               method=torch.empty(B, T, dtype=torch.uint8, device=dev),
               k_est=torch.empty(B, T, dtype=torch.int32, device=dev),
               info=torch.empty(B, T, dtype=torch.int32, device=dev),
               consumed=torch.zeros(B, dtype=torch.int64, device=dev),
               G_last=torch.empty(B, K, K, dtype=torch.complex128, device=dev),
               A_inv=(torch.empty(B, T, K, K, dtype=torch.complex128, device=dev)
                      if keep_A_inv else None))
    ws = workspace(dev, lib.lrz_trajectory_ws(_dt(H), B, T, K, Nn, D), "fused_traj")
    N.check(lib.lrz_trajectory(_dt(H), B, T, K, Nn, H.data_ptr(), float(alpha), float(P_t),
                               noise.data_ptr(), int(t0), int(n_reset),
                               C.byref(cfg) if cfg is not None else None,
                               N.ptr(omega), omega.stride(0) if omega is not None else 0,
                               A_inv_state.data_ptr(), N.ptr(A_state), N.ptr(G_prev),
                               out["G_last"].data_ptr(), out["rates"].data_ptr(),
                               out["per_ut"].data_ptr(), out["method"].data_ptr(),
                               out["k_est"].data_ptr(), out["info"].data_ptr(),
                               out["consumed"].data_ptr(), N.ptr(out["A_inv"]), ws.data_ptr(),
                               N.stream_ptr(dev)), "lrz_trajectory")
    _count(10)
    return out


def campaign_summary(rates: torch.Tensor, stats: torch.Tensor):
    """lrz_campaign_summary: rates [M,B,T] f64, stats [M,B,6] f64 (device) ->
    (trial_mean [M,B], summary [M,6], table [M,2]) on the device."""
    _chk(rates, "rates")
    _chk(stats, "stats")
    M, B, T = rates.shape
    dev = rates.device
    tm = torch.empty(M, B, dtype=torch.float64, device=dev)
    sm = torch.empty(M, 6, dtype=torch.float64, device=dev)
    tb = torch.empty(M, 2, dtype=torch.float64, device=dev)
    lib = N.lib_for(dev)
    N.check(lib.lrz_campaign_summary(M, B, T, rates.data_ptr(), stats.data_ptr(), tm.data_ptr(),
                                     sm.data_ptr(), tb.data_ptr(), N.stream_ptr(dev)),
            "lrz_campaign_summary")
    _count(2)
    return tm, sm, tb
