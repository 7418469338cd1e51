"""Host-side Gaussian sketch streams (Omega) for the device arSVD.

The reference draws each sketch inside ``arsvd`` from the caller's
``np.random.Generator`` as sqrt(1/2) * (N(K x d) + j N(K x d)), real block
first, both row-major (``lowrank.py:284-286``), and the harness shares one
Generator per (method, trial) across all time steps (``harness.py:206-211,
236-237``).  Because ``Generator.standard_normal`` is chunking-invariant
(the n-th normal does not depend on how the draws were batched), one flat
float64 normal stream per trial plus a device-side cursor reproduces the
reference's Omega bit for bit: an arSVD iteration of width d starting at
cursor c reads the real block at [c, c + K d) and the imaginary block at
[c + K d, c + 2 K d), then advances the cursor by 2 K d.

Consumption is data dependent (it depends on the number of arSVD
iterations), so each trial keeps a FIFO: normals are generated ahead in
chunks, the device reports the cursor it reached, and consumed normals
are dropped.
"""

from __future__ import annotations

import numpy as np

from .scenario import method_label, stream_seed


def sketch_widths(K: int, k_init: int, p: int, i_max: int) -> list[int]:
    """Widths d_i = min(k0_i + p, K), k0_i = k_init * 2^i (lowrank.py:279-302)."""
    out, k0 = [], k_init
    for _ in range(i_max):
        out.append(min(k0 + p, K))
        k0 *= 2
    return out


def normals_per_call_max(K: int, k_init: int, p: int, i_max: int) -> int:
    """Upper bound on normals one arsvd call consumes (all i_max iterations)."""
    return sum(2 * K * d for d in sketch_widths(K, k_init, p, i_max))


def effective_i_max(K: int, k_init: int, p: int, i_max: int, eta_max: float) -> int:
    """Iterations an arsvd call can actually run.  Once the sketch width
    reaches K the basis Q is a full unitary (Householder QR), so B = Q^H dA
    keeps all of ||dA||_F^2 and the energy rule (lowrank.py:290-301) is met
    for any eta below 1 - 1e-9: the loop never goes past that iteration."""
    if eta_max > 1.0 - 1e-9:
        return i_max
    k0 = k_init
    for i in range(i_max):
        if min(k0 + p, K) == K:
            return i + 1
        k0 *= 2
    return i_max


def normals_per_call_bound(K: int, k_init: int, p: int, i_max: int, eta_max: float) -> int:
    """Upper bound on normals one call consumes at energy fractions <= eta_max."""
    i_eff = effective_i_max(K, k_init, p, i_max, eta_max)
    return sum(2 * K * d for d in sketch_widths(K, k_init, p, i_eff))


def consumed_by(iters: np.ndarray, K: int, k_init: int, p: int, i_max: int) -> np.ndarray:
    """Normals consumed by a call that ran ``iters`` iterations (0 = none)."""
    cum = np.concatenate([[0], np.cumsum([2 * K * d for d in
                                          sketch_widths(K, k_init, p, i_max)])])
    return cum[np.asarray(iters, dtype=np.int64)]


class OmegaStreams:
    """One sequential standard-normal stream per trial.

    ``window(n)`` returns a (B, n) float64 array whose row b starts at that
    trial's first unconsumed normal; ``advance(consumed)`` drops the
    normals a device pass consumed.  The same object drives the oracle
    (``oracle/``) and the GPU path, so both see identical sketches.
    """

    def __init__(self, generators):
        self._gens = list(generators)
        self._buf = [np.empty(0) for _ in self._gens]
        self.consumed_total = np.zeros(len(self._gens), dtype=np.int64)

    @classmethod
    def for_method(cls, master_seed: int, eta: float, trials) -> "OmegaStreams":
        """Streams keyed exactly like the reference harness's per-(method,
        trial) sketch Generator (harness.py:88-92,206-211)."""
        label = method_label(eta)
        return cls(np.random.default_rng(stream_seed(master_seed, label, t)) for t in trials)

    @property
    def B(self) -> int:
        return len(self._gens)

    def _fill(self, b: int, n: int) -> None:
        have = self._buf[b].size
        if have < n:
            extra = self._gens[b].standard_normal(max(n - have, 1 << 12))
            self._buf[b] = np.concatenate([self._buf[b], extra])

    def window(self, n: int, out: np.ndarray | None = None) -> np.ndarray:
        """(B, n) block of the next n unconsumed normals of every trial."""
        if out is None:
            out = np.empty((self.B, n), dtype=np.float64)
        for b in range(self.B):
            self._fill(b, n)
            out[b] = self._buf[b][:n]
        return out

    def advance(self, consumed) -> None:
        consumed = np.broadcast_to(np.asarray(consumed, dtype=np.int64), (self.B,))
        for b in range(self.B):
            c = int(consumed[b])
            self._fill(b, c)
            self._buf[b] = self._buf[b][c:]
        self.consumed_total += consumed


class GeneratorBudget:
    """Adapter for the single-call API, which receives a bare
    ``np.random.Generator`` like the reference's ``arsvd(dA, cfg, rng)``.

    Draws a worst-case block from a snapshot of the generator state, and
    after the device reports how many normals it used, rewinds and redraws
    exactly that many so the caller's generator ends in the same state as
    after the reference call."""

    def __init__(self, rng: np.random.Generator, n_max: int):
        self.rng = rng
        self._state = rng.bit_generator.state
        self.block = rng.standard_normal(n_max)

    def commit(self, consumed: int) -> None:
        self.rng.bit_generator.state = self._state
        if consumed:
            self.rng.standard_normal(int(consumed))


def _split_u128(x: int) -> tuple[int, int]:
    return x & 0xFFFFFFFFFFFFFFFF, x >> 64


class DeviceOmegaStreams:
    """The same per-trial sketch streams as ``OmegaStreams``, generated on the
    GPU (``lrz_rng_normals``: PCG64 + numpy's ziggurat) from each Generator's
    PCG64 state, so neither host RNG time nor the Omega upload appears in the
    step.  ``window(L)`` -> device tensor [B, L]; ``advance(consumed)`` moves
    each stream past exactly the normals a device pass consumed (device
    tensor or array)."""

    def __init__(self, generators, device):
        import torch
        from . import _native as Nn, ops
        self._torch, self._N, self._ops = torch, Nn, ops
        self.device = torch.device(device)
        st, inc = [], []
        for g in generators:
            s = g.bit_generator.state
            if s.get("bit_generator") != "PCG64":
                raise TypeError("device streams reproduce PCG64 Generators only")
            st.extend(_split_u128(int(s["state"]["state"])))
            inc.extend(_split_u128(int(s["state"]["inc"])))
        as_u64 = lambda v: torch.tensor(np.array(v, dtype=np.uint64).view(np.int64),
                                        dtype=torch.int64, device=self.device)
        self.B = len(st) // 2
        self.state = as_u64(st).reshape(self.B, 2)
        self.inc = as_u64(inc).reshape(self.B, 2)
        self.raw = torch.zeros(self.B, dtype=torch.int64, device=self.device)
        self.consumed_total = torch.zeros(self.B, dtype=torch.int64, device=self.device)
        self._L = None
        self._ws = None        # this stream set's own RNG workspace (window tables)
        self.ready = None      # event of the last window generated on a side stream
        self._out = None       # reused window buffer

    @classmethod
    def for_method(cls, master_seed: int, eta: float, trials, device) -> "DeviceOmegaStreams":
        label = method_label(eta)
        return cls((np.random.default_rng(stream_seed(master_seed, label, t)) for t in trials),
                   device)

    def window(self, n: int, out=None, stream=None):
        """(B, n) device tensor of each trial's next n normals (a view of a
        buffer the next window() call overwrites).  With `stream`
        the generation runs there (after the current stream's pending work)
        and ``self.ready`` is an event the consumer waits on -- the RNG is
        integer work and overlaps the FP64 Gram stage."""
        torch = self._torch
        if stream is not None:
            cur = torch.cuda.current_stream(self.device)
            stream.wait_stream(cur)
            with torch.cuda.stream(stream):
                w = self.window(n, out)
                self.ready = torch.cuda.Event()
                self.ready.record(stream)
            if not torch.cuda.is_current_stream_capturing():
                w.record_stream(cur)
                self._ws.record_stream(cur)
            return w
        self.ready = None
        L = int(n)
        lib = self._N.lib_for(self.device)
        # one output buffer per stream set, reused by every window (the previous
        # window is dead once the next is requested: callers consume a window
        # within its chunk); avoids a multi-hundred-MB allocation per chunk
        if self._out is None or self._out.numel() < self.B * L:
            self._out = torch.empty(self.B * L, dtype=torch.float64, device=self.device)
        full = self._out[:self.B * L].view(self.B, L)
        status = torch.zeros(self.B, dtype=torch.int32, device=self.device)
        nbytes = int(lib.lrz_workspace_bytes(self._N.WS_RNG, 0, self.B, 0, L, 0))
        if self._ws is None or self._ws.numel() < nbytes:
            self._ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        self._N.check(lib.lrz_rng_normals(self.B, L, self.state.data_ptr(), self.inc.data_ptr(),
                                          self.raw.data_ptr(), full.data_ptr(), None,
                                          status.data_ptr(), self._ws.data_ptr(),
                                          self._N.stream_ptr(self.device)),
                      "lrz_rng_normals")
        self._status = status
        self._L = L
        self._ops._count(3)
        return full if out is None else out.copy_(full)

    def advance(self, consumed) -> None:
        """Skip exactly the first consumed[b] normals of the last window."""
        torch = self._torch
        c = torch.as_tensor(consumed, dtype=torch.int64, device=self.device).reshape(self.B)
        c = c.contiguous()
        adv = torch.empty(self.B, dtype=torch.int64, device=self.device)
        lib = self._N.lib_for(self.device)
        self._N.check(lib.lrz_rng_locate(self.B, self._L, self.state.data_ptr(),
                                         self.inc.data_ptr(), self.raw.data_ptr(), c.data_ptr(),
                                         adv.data_ptr(), self._ws.data_ptr(),
                                         self._N.stream_ptr(self.device)), "lrz_rng_locate")
        self._ops._count(1)
        self.raw += adv
        self.consumed_total += c
