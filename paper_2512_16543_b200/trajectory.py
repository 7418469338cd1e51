"""Batched trajectory runner: the B200 replacement of the reference's
per-trial sweep loop (harness._sweep_trial, harness.py:188-257).

For B Monte-Carlo trials x T time steps it produces, per (trial, step), the
maintained inverse A^-1_t, the precoder W_t = H_t^H A^-1_t (power
normalised) and the sum-rate, with the reference's step semantics:

* step 0 and every n_reset-th step: full inversion of the Gram
  (harness.py:229-233);
* conventional method: full inversion every step;
* WB-arSVD: arSVD of the Gram correction between consecutive channels
  (harness.py:234-241) and the rank-ratio dispatcher (lowrank.py:345-373).

Execution plan per time chunk (all device-resident, stream-ordered):

  1. G[b,t]  = H H^H + alpha I            batched over B*T       (K1)
  2. dG[b,t] = gram_delta(H_{t-1}, H_t)    batched over B*T       (K1')
  3. arSVD of every dG with *speculative* sketch cursors, batched over
     B*T; a verifier re-runs only the steps whose cursor was mispredicted
     (the sketch stream is the only thing that serialises arSVD across
     steps, and iteration counts rarely change between passes)  (K2+K3)
  4. plan[b,t] = full / woodbury / none   (dispatcher, lowrank.py:345-359)
  5. inv(G) for every full step           batched over B*T        (K5)
  6. Woodbury recurrence per trial        sequential in t only    (K4)
  7. precoder + SINR / sum-rate           batched over B*T        (K6)
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import ops
from .errors import SingularMatrixError
from .lowrank import cost_full, cost_wb_arsvd, sketch_cost
from .omega import OmegaStreams, consumed_by, effective_i_max, normals_per_call_bound


@dataclass
class TrajectoryConfig:
    """Method and knobs.  eta None = conventional (full inversion every step)."""

    alpha: float
    P_t: float = 1.0
    eta: float | None = None     # or a sequence: one eta per trial
    k_init: int = 2
    p: int = 5
    i_max: int = 3
    n_reset: int = 1200          # config.py:59
    maintain_A: bool = True      # keep A = A + U S V^H like GramState.A (lowrank.py:220)
    # speculative (batched over all steps) arSVD passes before the remaining
    # unverified suffixes are resolved in order (lrz_arsvd_seq)
    spec_passes: int = 2
    # H W for the rate from the Gram: (G - alpha I) A^-1 (exact with F_RF = I)
    rate_via_gram: bool = True
    # Gram correction: "diff" = G_t - G_{t-1} from the Grams already formed (complex128:
    # cancellation error ~1e-14 relative); "formula" = the gram_delta products; "auto" =
    # diff when the Grams are fp64-accumulated (complex128, or complex64 on the
    # FP64 tensor pipe), formula otherwise (complex64 FP32 Grams)
    delta: str = "auto"
    # resolve the sketch cursors with the energy-screen walk (lrz_arsvd_walk, K <= 32)
    # before the first speculative pass: True / False, or None = when eta < 0.99
    # (ranks then usually hit before the iteration cap, so iteration counts follow
    # the sketch and a first speculative pass at predicted cursors is wasted)
    walk_first: bool | None = None
    # screen-only cursor-resolution rounds run by that walk before the in-order
    # kernel: -1 = 16 (an idle round costs ~40 us; C2 at eta = 0.9 needs up to ~12:
    # a trial's borderline steps settle one per round), 0 = none (warp walk only)
    screen_rounds: int = -1


@dataclass
class ChunkResult:
    rates: torch.Tensor          # [B, T] sum-rate
    per_ut: torch.Tensor         # [B, T, K]
    method: torch.Tensor         # [B, T] uint8 (full 0, woodbury 1, none 2)
    k_est: torch.Tensor          # [B, T] int32 (0 on full-reset steps)
    iters: torch.Tensor          # [B, T] int32 arSVD iterations
    info: torch.Tensor           # [B, T] int32 kernel status
    A_inv: torch.Tensor | None   # [B, T, K, K] complex128
    W: torch.Tensor | None       # [B, T, N, K] unscaled F_raw
    scale: torch.Tensor          # [B, T] power normalisation
    consumed: torch.Tensor       # [B] normals consumed in this chunk
    spec_passes: int = 0
    flags: torch.Tensor | None = None   # sync=False: [unverified trials, short windows]


@dataclass
class TrajectoryResult:
    rates: np.ndarray
    per_ut: np.ndarray
    method: np.ndarray
    k_est: np.ndarray
    iters: np.ndarray
    cost: np.ndarray
    consumed: np.ndarray
    spec_passes: list = field(default_factory=list)
    A_inv: np.ndarray | None = None
    W: np.ndarray | None = None          # [B, T, N, K] power-normalised precoder F_BB
    scale: np.ndarray | None = None      # [B, T] power normalisation s (F_BB = s F_raw)


_MASKS: dict = {}   # dispatcher-step masks by (B, reset pattern, device)


class _nullctx:
    def __enter__(self):
        return None

    def __exit__(self, *a):
        return False
_PINNED: list = []  # one pinned int32[2] readback buffer (page-locking per call is slow)


def _pinned_flags() -> torch.Tensor:
    if not _PINNED:
        _PINNED.append(torch.zeros(2, dtype=torch.int32).pin_memory())
    return _PINNED[0]


class TrajectoryRunner:
    """Stateful runner over consecutive time chunks of B trials."""

    def __init__(self, B: int, K: int, N: int, dtype: torch.dtype, cfg: TrajectoryConfig,
                 device=None):
        self.B, self.K, self.N, self.dtype, self.cfg = B, K, N, dtype, cfg
        self.device = torch.device(device) if device is not None else torch.device("cuda", 0)
        self.t = 0
        self.H_prev = None
        self.G_prev = None
        self.A_inv = torch.zeros(B, K, K, dtype=torch.complex128, device=self.device)
        self.A = torch.zeros(B, K, K, dtype=torch.complex128, device=self.device)
        self.D = ops.d_max_for(K, cfg.k_init, cfg.p, cfg.i_max)
        # eta: None (conventional), a float, or one value per trial (several WB
        # methods batched as trials of one runner)
        self._eta = cfg.eta
        if cfg.eta is not None and np.ndim(cfg.eta) == 1:
            e = np.asarray(cfg.eta, dtype=np.float64)
            if e.shape != (B,) or not np.all((e > 0) & (e <= 1)):
                raise ValueError("per-trial eta must have one value in (0, 1] per trial")
            self._eta = torch.from_numpy(e).to(self.device)
        self.prof = None          # list of (stage, start_event, end_event) when profiling
        self._in_order = False    # set once a chunk needed the in-order arSVD
        self._walk_first = False  # set once a chunk needed the cursor walk

    def snapshot(self) -> dict:
        """Copy of the chunk-to-chunk state (for re-running a sync=False chunk)."""
        cl = lambda x: None if x is None else x.clone()  # noqa: E731
        return dict(t=self.t, H_prev=cl(self.H_prev), G_prev=cl(self.G_prev),
                    A_inv=self.A_inv.clone(), A=self.A.clone(), in_order=self._in_order,
                    walk_first=self._walk_first)

    def restore(self, snap: dict) -> None:
        self.t, self.H_prev, self.G_prev = snap["t"], snap["H_prev"], snap["G_prev"]
        self.A_inv.copy_(snap["A_inv"])
        self.A.copy_(snap["A"])
        self._in_order, self._walk_first = snap["in_order"], snap["walk_first"]

    def _ev(self):
        if self.prof is None:
            return None
        e = torch.cuda.Event(enable_timing=True)
        e.record(torch.cuda.current_stream(self.device))
        return e

    def _stage(self, name, e0):
        if self.prof is not None:
            self.prof.append((name, e0, self._ev()))

    # -- helpers -------------------------------------------------------------
    def _eta_max(self) -> float:
        return float(np.max(np.asarray(self.cfg.eta, dtype=np.float64)))

    def normals_per_step_max(self) -> int:
        """Window normals one step may need (see omega.effective_i_max)."""
        c = self.cfg
        return 0 if c.eta is None else normals_per_call_bound(self.K, c.k_init, c.p, c.i_max,
                                                              self._eta_max())

    def _is_sketch(self, T: int):
        """(device [B, T] uint8 mask of dispatcher steps, host count per trial);
        built on the host from the step indices -- no device round trip."""
        c = self.cfg
        tg = np.arange(self.t, self.t + T)
        reset = (tg == 0) | ((c.n_reset > 0) & (tg % max(c.n_reset, 1) == 0))
        if self.H_prev is None:
            reset[0] = True
        if c.eta is None:
            reset[:] = True
        key = (self.B, reset.tobytes(), self.device)
        dev_mask = _MASKS.get(key)
        if dev_mask is None:
            row = torch.from_numpy((~reset).astype(np.uint8))
            dev_mask = row.to(self.device).reshape(1, T).expand(self.B, T).contiguous()
            if len(_MASKS) > 64:
                _MASKS.clear()
            _MASKS[key] = dev_mask
        return dev_mask, int((~reset).sum())

    def _tail(self, G, Hf, noise, is_sketch, iters_pred, cursor, res, k_est, plan, hybrid,
              keep_W, precode_stream=None):
        """Stages 4-7 of a chunk (dispatcher, batched full inversions, Woodbury
        chain, precoder + rate) from the arSVD results.  precode_stream: stage 7
        (the throughput-bound products W = H^H A^-1 and the coupling) is queued
        on that stream behind an event; stages 4-6 stay on the current one."""
        c = self.cfg
        B, T, K = G.shape[0], G.shape[1], self.K
        BT, Nn, dev = B * T, Hf.shape[-1], self.device
        iters = torch.zeros(B, T, dtype=torch.int32, device=dev)
        consumed = torch.zeros(B, dtype=torch.int64, device=dev)
        if res is not None:
            iters.copy_(iters_pred * is_sketch.to(torch.int32))
            U, V, S = res["U"], res["V"], res["S"]
            consumed = cursor[:, -1] + res["consumed"].reshape(B, T)[:, -1] * is_sketch[:, -1]
            # 4. dispatcher
            ops.plan(is_sketch, k_est, K, out=plan)
        else:
            U = torch.zeros(BT, 1, K, dtype=torch.complex128, device=dev)
            V = torch.zeros_like(U)
            S = torch.ones(BT, 1, dtype=torch.float64, device=dev)
        # 5. full inversions (plan == 0) batched
        A_inv_seq = torch.empty(B, T, K, K, dtype=torch.complex128, device=dev)
        info = torch.zeros(B, T, dtype=torch.int32, device=dev)
        full_mask = (plan == 0).to(torch.uint8)
        e0 = self._ev()
        ops.herm_inverse(G.reshape(BT, K, K), 1e14, mask=full_mask.reshape(BT),
                         out=A_inv_seq.reshape(BT, K, K), info=info.reshape(BT))
        self._stage("inverse", e0)
        # 6. sequential Woodbury recurrence per trial
        method = torch.zeros(B, T, dtype=torch.uint8, device=dev)
        e0 = self._ev()
        # K > 64: the step-parallel chain (products batched over trials) when there are
        # dispatcher steps; up to K = 64 one CTA per trial with the trial's A^-1
        # resident in shared memory (the step's products on DMMA)
        ops.chain(plan, G, self.A_inv, A_inv_seq, self.A if c.maintain_A else None, U, V, S,
                  k_est, method, info, steps=(res is not None and K > 64))
        self._stage("chain", e0)
        # 7. precoder and rate
        e0 = self._ev()
        ctx = _nullctx()
        if precode_stream is not None:
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(dev))
            precode_stream.wait_event(ev)
            used = [G, Hf, noise, A_inv_seq]
            if hybrid is not None:
                used.extend(v for v in hybrid.values() if isinstance(v, torch.Tensor))
            for t_ in used:
                t_.record_stream(precode_stream)
            ctx = torch.cuda.stream(precode_stream)
        with ctx:
            pr, W = self._precode(G, Hf, noise, A_inv_seq, hybrid, keep_W, T)
        self._stage("precode_rate", e0)
        return A_inv_seq, method, info, pr, W, iters, consumed

    def _precode(self, G, Hf, noise, A_inv_seq, hybrid, keep_W, T):
        c = self.cfg
        K, dev = self.K, self.device
        BT, Nn = Hf.shape[0], Hf.shape[-1]
        if hybrid is not None:
            pr = ops.hybrid_precode_rate(Hf, A_inv_seq.reshape(BT, K, K),
                                         hybrid["H_rf"].reshape(BT, K, Nn),
                                         hybrid["cols"].reshape(BT, Nn), hybrid["n_x"],
                                         hybrid["n_y"], hybrid["dft"], c.P_t, noise, T,
                                         want_F=keep_W)
            W = pr["F_BB"]
        else:
            W = torch.empty(BT, Nn, K, dtype=self.dtype, device=dev) if keep_W else None
            pr = ops.precode_rate(Hf, A_inv_seq.reshape(BT, K, K), c.P_t, noise, T, W=W,
                                  want_sinr=False,
                                  G_true=G.reshape(BT, K, K) if c.rate_via_gram else None,
                                  alpha=c.alpha)
        return pr, W

    def gram_async(self, H: torch.Tensor, heavy_stream):
        """Stage 1 of a chunk (the true Grams) queued on ``heavy_stream`` behind
        the current stream's work so far; returns (G, event) for
        ``run_chunk(gram=...)``.  The pipelined caller issues chunk c + 1's Grams
        before ``run_chunk`` of chunk c, so that they precede chunk c's precoder
        on the heavy stream."""
        B, T, K, Nn = H.shape
        cur = torch.cuda.current_stream(self.device)
        ev = torch.cuda.Event()
        ev.record(cur)
        heavy_stream.wait_event(ev)
        H.record_stream(heavy_stream)
        with torch.cuda.stream(heavy_stream):
            G = ops.gram(H.reshape(B * T, K, Nn), self.cfg.alpha).reshape(B, T, K, K)
            done = torch.cuda.Event()
            done.record(heavy_stream)
        G.record_stream(cur)
        return G, done

    def _tail_on(self, stream, G, Hf, noise, is_sketch, *rest):
        """_tail on `stream` after the current stream's work so far; the
        tensors it reads are marked as used there (allocator safety)."""
        cur = torch.cuda.current_stream(self.device)
        ev = torch.cuda.Event()
        ev.record(cur)
        stream.wait_event(ev)
        used = [G, Hf, noise, is_sketch]
        for x in rest:
            if isinstance(x, torch.Tensor):
                used.append(x)
            elif isinstance(x, dict):
                used.extend(v for v in x.values() if isinstance(v, torch.Tensor))
        for t_ in used:
            t_.record_stream(stream)
        with torch.cuda.stream(stream):
            return self._tail(G, Hf, noise, is_sketch, *rest)

    # -- one chunk -------------------------------------------------------------
    def run_chunk(self, H: torch.Tensor, noise: torch.Tensor, omega: torch.Tensor | None = None,
                  keep_A_inv: bool = False, keep_W: bool = False, hybrid: dict | None = None,
                  omega_ready=None, sync: bool = True, back_stream=None,
                  heavy_stream=None, gram=None) -> ChunkResult:
        """H [B, T, K, N] (device, self.dtype); noise [B, K] float64 (device);
        omega [B, L] float64 (device; row b = trial b's next unconsumed normals,
        L >= T * normals_per_step_max()).

        hybrid (analog beams, reference precoding.py:37-80 with F_RF != I): H is
        the effective channel H_eff = H~ F_RF and the dict carries H_rf = H F_RF
        [B,T,K,N_RF], cols [B,T,N_RF] (DFT codebook indices), n_x, n_y and dft
        (the two DFT factors) for the hybrid precoder / rate.  omega_ready: CUDA
        event the sketch window was produced under (another stream).

        sync=False: no host round trip at all (CUDA-graph capture): the chunk is
        computed optimistically from the first arSVD pass and ``result.flags``
        (device int32[2]: unverified trials, short sketch windows) must be
        checked by the caller.  Nonzero means the results are not the
        reference's: the runner's state (t, H_prev, G_prev, A_inv, A) has
        already advanced past this chunk, so the re-run with sync=True needs a
        FRESH runner (or one restored with ``snapshot()`` / ``restore()`` taken
        before the call) and the same sketch window.

        back_stream (with sync=False): stages 4-7 (dispatcher, inversions,
        Woodbury chain, precoder + rate) run on that stream behind an event,
        while the current stream returns to the caller for the next chunk's
        Grams and arSVD -- the latency-bound chain of chunk c overlaps the
        throughput-bound products of chunk c + 1.  The next chunk's front
        stages depend only on this chunk's front stages (last Gram, sketch
        consumption), the chain only on the previous chain (same stream).
        The caller joins ``back_stream`` before reading the results.

        heavy_stream (with sync=False; instead of back_stream): the two
        throughput-bound stages -- the Grams (stage 1) and the precoder products
        (stage 7), both at the FP64 tensor-pipe peak from K = 64 -- are queued on
        that (low-priority) stream, everything between them (Gram corrections,
        arSVD, inversions, chain: latency-bound launches) stays on the current
        stream, which the caller gives the higher priority.  With
        ``gram=self.gram_async(H_next, heavy_stream)`` issued before this call the
        heavy stream runs  G(c+1) | W(c) | G(c+2) | W(c+1) ...  back to back while
        the light stages of chunk c + 1 run beside W(c) on the SMs' spare
        registers.  The caller joins ``heavy_stream`` before reading rates / W."""
        c = self.cfg
        B, T, K, Nn = H.shape
        assert (B, K, Nn) == (self.B, self.K, self.N) and H.dtype == self.dtype
        dev = self.device
        BT = B * T
        Hf = H.reshape(BT, K, Nn)
        is_sketch, n_sketch = self._is_sketch(T)

        if heavy_stream is not None:
            assert not sync and back_stream is None
        # 1. true Grams of every step
        e0 = self._ev()
        if heavy_stream is not None:
            G, g_ready = gram if gram is not None else self.gram_async(H, heavy_stream)
            assert G.shape == (B, T, K, K)
            torch.cuda.current_stream(dev).wait_event(g_ready)
        else:
            G = ops.gram(Hf, c.alpha).reshape(B, T, K, K)
        self._stage("gram", e0)
        plan = torch.zeros(B, T, dtype=torch.uint8, device=dev)
        k_est = torch.zeros(B, T, dtype=torch.int32, device=dev)
        D = self.D
        passes = 0
        chunk_flags = None
        if n_sketch:
            # 2. Gram corrections between consecutive channels (dH = H_t - H_{t-1})
            dA = torch.empty(B, T, K, K, dtype=torch.complex128, device=dev)
            dAf = dA.reshape(BT, K, K)
            e0 = self._ev()
            # "auto": difference the complex128 Grams whenever they are accumulated in
            # fp64 -- complex128 inputs, or complex64 H widened to fp64 on the tensor
            # pipe (gram_dmma_kernel)
            fp64_gram = self.dtype == torch.complex128 or ops.dmma_active()
            use_diff = c.delta == "diff" or (c.delta == "auto" and fp64_gram)
            if use_diff:
                Gf = G.reshape(BT, K, K)
                if T > 1:
                    ops.axpby(1.0, Gf[1:], -1.0, Gf[:-1], out=dAf[1:])
                if self.G_prev is not None:
                    d0 = ops.axpby(1.0, G[:, 0].contiguous(), -1.0, self.G_prev)
                    dA[:, 0].copy_(d0)
            else:
                if T > 1:
                    ops.gram_delta(Hf[:-1], Hf[1:], 1, out=dAf[1:])
                if self.H_prev is not None:
                    ops.gram_delta(self.H_prev, H[:, 0], 1, out=dA[:, 0])
            self._stage("gram_delta", e0)
            # 3. speculative arSVD
            assert omega is not None and omega.shape[0] == B
            if omega_ready is not None:
                torch.cuda.current_stream(dev).wait_event(omega_ready)
            i_eff = effective_i_max(K, c.k_init, c.p, c.i_max, self._eta_max())
            iters_pred = torch.full((B, T), i_eff, dtype=torch.int32, device=dev)
            cursor = torch.zeros(B, T, dtype=torch.int64, device=dev)
            cursor0 = torch.zeros(B, dtype=torch.int64, device=dev)
            first = torch.zeros(B, dtype=torch.int32, device=dev)
            active = torch.zeros(B, T, dtype=torch.uint8, device=dev)
            pending = torch.zeros(1, dtype=torch.int32, device=dev)
            ops.spec_verify(is_sketch, iters_pred, None, cursor, cursor0, first, active, pending,
                            K, self._eta, c.k_init, c.p, c.i_max)
            row = torch.arange(B, dtype=torch.int32, device=dev).repeat_interleave(T)
            res = dict(
                U=torch.empty(BT, D, K, dtype=torch.complex128, device=dev),
                V=torch.empty(BT, D, K, dtype=torch.complex128, device=dev),
                S=torch.zeros(BT, D, dtype=torch.float64, device=dev),
                k_est=k_est.reshape(BT),
                iters=torch.zeros(BT, dtype=torch.int32, device=dev),
                fallback=torch.zeros(BT, dtype=torch.int32, device=dev),
                consumed=torch.zeros(BT, dtype=torch.int64, device=dev),
            )
            n_spec = 0 if self._in_order else c.spec_passes
            # cursor walk (K <= 32): resolves every step's cursor from the energy
            # screen alone, in order, so one more speculative pass settles the chunk
            walk_kernel = ops.walk_ok(K, c.k_init, c.p, c.i_max)
            can_screen = D <= 40 and c.screen_rounds != 0
            can_walk = n_spec > 0 and (walk_kernel or can_screen)

            def walk():
                e0 = self._ev()
                first0 = first.clone()   # steps before it hold verified exact factors
                if can_screen:
                    # screen-only rounds, batched over every unsettled step: each round
                    # takes the iteration counts the CholeskyQR energy screen sees at
                    # the current cursors, accepts every trial's prefix up to its first
                    # changed count and re-bases the cursors behind it (no host sync)
                    rounds = c.screen_rounds if c.screen_rounds > 0 else 16
                    # counts that hinge on the sketch drawn are not carried over from a
                    # pass at shifted cursors: the suffix is re-predicted by majority
                    votes = torch.empty(B, T, ops.SPEC_VOTE_W, dtype=torch.uint8, device=dev)
                    pending.zero_()
                    ops.spec_verify(is_sketch, iters_pred, None, cursor, cursor0, first, active,
                                    pending, K, self._eta, c.k_init, c.p, c.i_max, votes=votes)
                    for _ in range(rounds):
                        ops.arsvd(dAf, omega, cursor.reshape(BT), self._eta, c.k_init, c.p,
                                  c.i_max, omega_row=row, mask=active.reshape(BT), out=res,
                                  want_factor=2, hermitian=True)
                        pending.zero_()
                        ops.spec_verify(is_sketch, iters_pred, res["iters"], cursor, cursor0,
                                        first, active, pending, K, self._eta, c.k_init, c.p,
                                        c.i_max, votes=votes)
                if walk_kernel:
                    # trials the rounds left unsettled (the kernel returns at once for
                    # the others): in order, one warp per trial
                    ops.arsvd_walk(dA, omega, is_sketch, first, cursor, iters_pred, self._eta,
                                   c.k_init, c.p, c.i_max)
                first.copy_(first0)
                pending.zero_()
                ops.spec_verify(is_sketch, iters_pred, None, cursor, cursor0, first, active,
                                pending, K, self._eta, c.k_init, c.p, c.i_max)
                self._stage("walk", e0)

            def one_pass():
                e0 = self._ev()
                if passes < n_spec:
                    ops.arsvd(dAf, omega, cursor.reshape(BT), self._eta, c.k_init, c.p, c.i_max,
                              omega_row=row, mask=active.reshape(BT), out=res,
                              want_factor=False, hermitian=True)
                else:
                    # iteration counts keep changing with the sketch: resolve the rest
                    # of every trial in order (one CTA per trial, exact cursors)
                    ops.arsvd_seq(dA, omega, is_sketch, first, cursor, iters_pred, self._eta,
                                  c.k_init, c.p, c.i_max, res)
                self._stage("arsvd", e0)
                pending.zero_()
                e0 = self._ev()
                ops.spec_verify(is_sketch, iters_pred, res["iters"], cursor, cursor0, first,
                                active, pending, K, self._eta, c.k_init, c.p, c.i_max)
                self._stage("verify", e0)
                # pending trials, and calls that found their sketch window too short
                torch.stack([pending[0], (res["iters"] < 0).sum().to(torch.int32)],
                            out=flags)

            flags = torch.zeros(2, dtype=torch.int32, device=dev)
            A_state0 = self.A.clone() if (c.maintain_A and sync) else None
            walked = False
            wf = c.walk_first if c.walk_first is not None else self._eta_max() < 0.99
            if can_walk and (self._walk_first or wf):
                walk()          # the last chunk's iteration counts followed the sketch
                walked = True
            one_pass()
            passes = 1
            # optimistic: the rest of the chunk is queued behind the first pass and
            # only then is the verifier's answer read back (one sync per chunk)
            if heavy_stream is not None:
                tail = self._tail(G, Hf, noise, is_sketch, iters_pred, cursor, res, k_est, plan,
                                  hybrid, keep_W, precode_stream=heavy_stream)
            elif back_stream is not None and not sync:
                # this chunk's sketch consumption, on the front stream (the next
                # chunk's window advance must not wait for the back stages)
                front_consumed = cursor[:, -1] + \
                    res["consumed"].reshape(B, T)[:, -1] * is_sketch[:, -1]
                tail = self._tail_on(back_stream, G, Hf, noise, is_sketch, iters_pred, cursor,
                                     res, k_est, plan, hybrid, keep_W)
                tail = tail[:-1] + (front_consumed,)
            else:
                tail = self._tail(G, Hf, noise, is_sketch, iters_pred, cursor, res, k_est, plan,
                                  hybrid, keep_W)
            chunk_flags = flags
            if sync:
                pinned = _pinned_flags()
                pinned.copy_(flags, non_blocking=True)
                torch.cuda.current_stream(dev).synchronize()
                if int(pinned[1]):
                    raise RuntimeError("sketch window shorter than an arsvd call needed")
                if int(pinned[0]):
                    while True:
                        if can_walk and not walked:
                            walk()
                            walked = True
                            self._walk_first = True
                        one_pass()
                        passes += 1
                        pinned.copy_(flags, non_blocking=True)
                        torch.cuda.current_stream(dev).synchronize()
                        if int(pinned[1]):
                            raise RuntimeError("sketch window shorter than an arsvd call needed")
                        if int(pinned[0]) == 0:
                            break
                        if passes > n_spec:
                            raise RuntimeError("in-order arSVD left unverified steps")
                    if A_state0 is not None:
                        self.A.copy_(A_state0)
                    tail = self._tail(G, Hf, noise, is_sketch, iters_pred, cursor, res, k_est,
                                      plan, hybrid, keep_W)
                if passes > n_spec:
                    self._in_order = True   # iteration counts track the sketch: skip speculation
        elif heavy_stream is not None:
            tail = self._tail(G, Hf, noise, is_sketch, None, None, None, k_est, plan, hybrid,
                              keep_W, precode_stream=heavy_stream)
        elif back_stream is not None and not sync:
            tail = self._tail_on(back_stream, G, Hf, noise, is_sketch, None, None, None, k_est,
                                 plan, hybrid, keep_W)
        else:
            tail = self._tail(G, Hf, noise, is_sketch, None, None, None, k_est, plan, hybrid,
                              keep_W)
        A_inv_seq, method, info, pr, W, iters, consumed = tail
        # state for the next chunk
        self.H_prev = H[:, -1].contiguous().clone()
        self.G_prev = G[:, -1].contiguous().clone()
        self.t += T
        bs = back_stream if (back_stream is not None and not sync) else None
        with torch.cuda.stream(bs) if bs is not None else _nullctx():
            self.A_inv = A_inv_seq[:, -1].clone()
        if heavy_stream is not None:
            bs = heavy_stream     # the precoder's status is produced there
            info.record_stream(heavy_stream)
        with torch.cuda.stream(bs) if bs is not None else _nullctx():
            # status per step: the inverse's code (singular / indefinite) wins over the
            # precoder's (zero norm), so a singular step is never hidden by a later code
            pinfo = pr["info"].reshape(B, T)
            info = torch.where(info != 0, info, pinfo)
        return ChunkResult(rates=pr["sum"].reshape(B, T), per_ut=pr["rates"].reshape(B, T, K),
                           method=method, k_est=k_est, iters=iters, info=info,
                           A_inv=A_inv_seq if keep_A_inv else None,
                           W=W.reshape(B, T, *W.shape[1:]) if keep_W else None,
                           scale=pr["scale"].reshape(B, T), consumed=consumed,
                           spec_passes=passes, flags=None if sync else chunk_flags)


def step_costs(method: np.ndarray, k_est: np.ndarray, is_sketch: np.ndarray, K: int) -> np.ndarray:
    """Cost units per step as the harness records them (harness.py:233,239):
    resets cost K^3; dispatcher full = K^3 + sketch; woodbury; none."""
    m = np.asarray(method)
    k = np.asarray(k_est).astype(float)
    sk = np.asarray(is_sketch, dtype=bool)
    Kf = float(K)
    full = cost_full(K)
    sketch = Kf ** 2 * k + k ** 2 * Kf                        # sketch_cost(K, k)
    wb = Kf ** 2 + Kf ** 2 * k + k ** 3 + k ** 2 * Kf         # cost_wb_arsvd(K, k)
    out = np.where(m == 0, full + sketch, np.where(m == 1, wb, cost_wb_arsvd(K, 0)))
    return np.where(sk, out, full).astype(float)


def run_trajectory(H, noise, cfg: TrajectoryConfig, streams: OmegaStreams | None = None,
                   chunk: int | None = None, keep_A_inv: bool = False,
                   device=None, keep_W: bool = False) -> TrajectoryResult:
    """Run B trials x T steps.  H: numpy or torch [B, T, K, N]; noise [K] or
    [B, K]; streams: per-trial sketch streams (required for WB): host
    ``OmegaStreams`` or GPU-generated ``DeviceOmegaStreams`` (same normals)."""
    dev = torch.device(device) if device is not None else (
        H.device if isinstance(H, torch.Tensor) and H.is_cuda else torch.device("cuda", 0))
    if isinstance(H, np.ndarray):
        tdt = torch.complex64 if H.dtype == np.complex64 else torch.complex128
    else:
        tdt = H.dtype
    B, T, K, Nn = H.shape
    chunk = T if chunk is None else chunk
    nz = np.array(np.broadcast_to(np.asarray(noise, dtype=np.float64), (B, K)), order="C")
    noise_d = torch.from_numpy(nz).to(dev)
    runner = TrajectoryRunner(B, K, Nn, tdt, cfg, dev)
    outs = []
    passes = []
    cons_total = np.zeros(B, dtype=np.int64)
    for t0 in range(0, T, chunk):
        t1 = min(T, t0 + chunk)
        Hc = H[:, t0:t1]
        Hc = (torch.from_numpy(np.ascontiguousarray(Hc)).to(dev) if isinstance(Hc, np.ndarray)
              else Hc.to(dev).contiguous())
        om = None
        if cfg.eta is not None:
            L = (t1 - t0) * runner.normals_per_step_max()
            om = streams.window(L)
            if isinstance(om, np.ndarray):  # host streams (OmegaStreams); device streams stay put
                om = torch.from_numpy(om).to(dev)
        r = runner.run_chunk(Hc, noise_d, om, keep_A_inv=keep_A_inv, keep_W=keep_W)
        if keep_W:
            # F_BB = s F_raw (precoding.py:47-52), moved to the host chunk by chunk
            r.W = (r.W * r.scale[..., None, None].to(r.W.dtype)).cpu()
        if cfg.eta is not None:
            used = r.consumed.cpu().numpy()
            streams.advance(r.consumed if isinstance(om, torch.Tensor) and
                            not isinstance(streams, OmegaStreams) else used)
            cons_total += used
        passes.append(r.spec_passes)
        outs.append(r)
    info = torch.cat([o.info for o in outs], 1).cpu().numpy()
    if np.any(info == 1):
        b, t = np.argwhere(info == 1)[0]
        raise SingularMatrixError(f"trial {b} step {t}: condition estimate exceeds 1e14")
    method = torch.cat([o.method for o in outs], 1).cpu().numpy()
    k_est = torch.cat([o.k_est for o in outs], 1).cpu().numpy()
    iters = torch.cat([o.iters for o in outs], 1).cpu().numpy()
    sk = iters > 0
    # steps that ran the dispatcher but consumed nothing (zero perturbation) still count
    tg = np.arange(T)
    sk_mask = np.broadcast_to((tg > 0) & ~((cfg.n_reset > 0) & (tg % max(cfg.n_reset, 1) == 0)),
                              (B, T)) if cfg.eta is not None else np.zeros((B, T), bool)
    cons = consumed_by(iters, K, cfg.k_init, cfg.p, cfg.i_max) if cfg.eta is not None else \
        np.zeros((B, T), np.int64)
    del sk
    return TrajectoryResult(
        rates=torch.cat([o.rates for o in outs], 1).cpu().numpy(),
        per_ut=torch.cat([o.per_ut for o in outs], 1).cpu().numpy(),
        method=method, k_est=k_est, iters=iters,
        cost=step_costs(method, k_est, sk_mask, K), consumed=cons, spec_passes=passes,
        A_inv=(torch.cat([o.A_inv for o in outs], 1).cpu().numpy() if keep_A_inv else None),
        W=(torch.cat([o.W for o in outs], 1).numpy() if keep_W else None),
        scale=torch.cat([o.scale for o in outs], 1).cpu().numpy())


def run_campaign_device(spec, eta, trials, device=None, chunk: int | None = None,
                        keep: bool = True) -> TrajectoryResult:
    """A whole synthetic pass for the given trials with everything on the
    GPU: channels synthesised per time chunk (``scenario.DeviceChannels``),
    sketches from the device RNG (``DeviceOmegaStreams``, the harness's
    per-(method, trial) streams), then the runner.  Only the per-step results
    come back to the host.  eta None = conventional method."""
    from . import scenario as S
    from .omega import DeviceOmegaStreams
    dev = torch.device(device) if device is not None else torch.device("cuda", 0)
    trials = list(trials)
    B, T, K, Nn = len(trials), spec.T, spec.K, spec.N
    chunk = T if chunk is None else chunk
    tdt = torch.complex64 if spec.dtype == "c64" else torch.complex128
    cfg = TrajectoryConfig(alpha=spec.alpha, eta=eta, k_init=spec.k_init, p=spec.p,
                           i_max=spec.i_max)
    chans = S.DeviceChannels(spec, trials, dev)
    streams = None if eta is None else DeviceOmegaStreams.for_method(spec.seed, eta, trials, dev)
    noise = torch.full((B, K), spec.noise_var, dtype=torch.float64, device=dev)
    runner = TrajectoryRunner(B, K, Nn, tdt, cfg, dev)
    outs, passes = [], []
    for t0 in range(0, T, chunk):
        t1 = min(T, t0 + chunk)
        H = chans.generate(t0, t1)
        om = None if eta is None else streams.window((t1 - t0) * runner.normals_per_step_max())
        r = runner.run_chunk(H, noise, om)
        if eta is not None:
            streams.advance(r.consumed)
        passes.append(r.spec_passes)
        if keep:
            outs.append({k: getattr(r, k).cpu() for k in ("rates", "per_ut", "method", "k_est",
                                                             "iters", "info")})
        del H
    if not keep:
        return None
    cat = {k: torch.cat([o[k] for o in outs], 1).numpy() for k in outs[0]}
    if np.any(cat["info"] == 1):
        b, t = np.argwhere(cat["info"] == 1)[0]
        raise SingularMatrixError(f"trial {trials[b]} step {t}: condition estimate exceeds 1e14")
    tg = np.arange(T)
    sk_mask = (np.broadcast_to((tg > 0) & ~((cfg.n_reset > 0) & (tg % max(cfg.n_reset, 1) == 0)),
                               (B, T)) if eta is not None else np.zeros((B, T), bool))
    cons = (consumed_by(cat["iters"], K, cfg.k_init, cfg.p, cfg.i_max) if eta is not None
            else np.zeros((B, T), np.int64))
    return TrajectoryResult(rates=cat["rates"], per_ut=cat["per_ut"], method=cat["method"],
                            k_est=cat["k_est"], iters=cat["iters"],
                            cost=step_costs(cat["method"], cat["k_est"], sk_mask, K),
                            consumed=cons, spec_passes=passes)
