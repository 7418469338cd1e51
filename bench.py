#!/usr/bin/env python
"""RZF precoder updates/s (WB-arSVD vs full inverse) and % of roofline on one B200
-- the BASELINE.json metric.

Headline workload (BASELINE.json configs[4], SURVEY.md 8(d) "C5", the largest
config whose channel tensor fits HBM): N = 4096 (64 x 64 UPA), K = 256 users,
T = 100 orbit steps, B = 64 Monte-Carlo trials per GPU, kappa 10 dB, drift
0.05 deg/step, SNR 10 dB (alpha = K / SNR), arSVD tolerance 1e-3 (eta =
0.999), rank cap 32 (i_max = 5), oversampling p = 5, complex128 (the
reference's own precision).  One bench "step" = one pass of the hot path over
the whole batch: B * T = 6,400 precoder updates, each producing A^-1_t, the
precoder W_t = H_t^H A^-1_t (written to HBM), its power normalisation and the
sum-rate (harness._sweep_trial semantics, harness.py:221-255; every C5 step
after the first is a rank-37 Woodbury update).  The channel tensor
H (107 GB) is resident in HBM before timing; the sketch normals are generated
on the device inside each step from the harness's per-(method, trial) PCG64
streams.

Beside the headline the line carries: the full-inversion method on the same
workload, per-kernel CUDA-event times over the timed region with the dominant
kernel's roofline, the end-to-end number through the public batched API with
host channels, and per-config keys for every other BASELINE config (C1, C2
c128/c64 incl. the paper's eta = 0.9 Woodbury regime, C3, the 12 C4 cap x tol
runs, C5 c64), each with its dominant-kernel roofline and CPU baseline.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--quick]

--impl reference times the reference algorithm on the host CPU (the numpy
oracle port of leorzf in oracle/, all cores, BLAS pinned to one thread per
worker like harness.py:284-293) on a bounded sample of the same workload.
Multi-GPU: torchrun, one rank per GPU, trials sharded by rank (weak scaling,
no data-path collective), max-over-ranks timing.
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "RZF precoder updates/s (WB-arSVD vs full inverse) and % of roofline, 1 B200"

# default T-chunk per config (HBM budget of the per-chunk working set)
CHUNK = {"C1": 50, "C2": 200, "C3": 50, "C4": 20, "C5": 20}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C5")
    ap.add_argument("--dtype", default="c128", choices=["c128", "c64"])
    ap.add_argument("--eta", type=float, default=None)
    ap.add_argument("--trials", type=int, default=None, help="trials per GPU (default: config B)")
    ap.add_argument("--T", type=int, default=None)
    ap.add_argument("--chunk", type=int, default=None)
    ap.add_argument("--e2e-trials", type=int, default=16)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline legs")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the per-config keys")
    ap.add_argument("--quick", action="store_true", help="per-config keys at reduced T")
    ap.add_argument("--pipe", default="back", choices=["auto", "heavy", "back", "off"],
                    help="stream schedules tried (auto: back, or heavy when > 3 %% faster)")
    return ap.parse_args()


def _spec(args):
    from paper_2512_16543_b200 import scenario as S
    spec = S.CONFIGS[args.config].with_(dtype=args.dtype)
    if args.trials:
        spec = spec.with_(B=args.trials)
    if args.T:
        spec = spec.with_(T=args.T)
    eta = spec.eta if args.eta is None else args.eta
    return spec, eta


def workload_desc(spec, eta):
    return (f"{spec.name}: N={spec.N} ({spec.n_side}x{spec.n_side} UPA), K={spec.K}, "
            f"T={spec.T}, B={spec.B} trials/GPU, SNR {spec.snr_db:g} dB, tol {1 - eta:.0e} "
            f"(eta={eta:g}), cap {spec.cap} (i_max={spec.i_max}), p={spec.p}, {spec.dtype}")


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# --------------------------------------------------------------------------- CPU legs

_BLAS_ENV = ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS",
             "SCIPY_OPENBLAS_NUM_THREADS")


def _cpu_init(spec_kw=None):
    """Worker initialiser: one BLAS thread (harness.py:284-293) and a short
    warm-up sweep so first-call library costs stay out of the timed trials."""
    try:
        import threadpoolctl
        threadpoolctl.threadpool_limits(1)
    except Exception:
        pass
    if spec_kw is not None:
        kw = dict(spec_kw)
        kw["T"] = 2
        _cpu_trial((kw, 0, 1.0 - kw["tol"], 2))


def _cpu_pool(cores, spec=None):
    """Spawned worker pool with BLAS pinned to one thread per process."""
    import multiprocessing as mp
    saved = {k: os.environ.get(k) for k in _BLAS_ENV}
    for k in _BLAS_ENV:
        os.environ[k] = "1"
    try:
        return mp.get_context("spawn").Pool(
            cores, initializer=_cpu_init,
            initargs=(dataclasses.asdict(spec) if spec is not None else None,))
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _cpu_trial(job):
    """The first `steps` steps of one trial of the reference algorithm (oracle
    port of lowrank/precoding through the _sweep_trial loop) on one core;
    channel generation is outside the timed region.  F_RF = I_N verbatim for
    N <= 1024, identity-elided at N = 4096."""
    spec_kw, trial, eta, steps = job
    from oracle import port, sweep
    from paper_2512_16543_b200 import scenario as S
    spec = S.ScenarioSpec(**spec_kw)
    H = S.trial_channels(spec, trial, 0, steps)
    if spec.dtype == "c64":
        H = H.astype(np.complex64)
    F = np.eye(spec.N) if spec.N <= 1024 else None
    cfg = None if eta is None else port.Cfg(eta, spec.k_init, spec.p, spec.i_max)
    sk = None if eta is None else np.random.default_rng(
        S.stream_seed(spec.seed, S.method_label(eta), trial))
    t0 = time.perf_counter()
    sweep.sweep_trial(H, spec.alpha, S.noise_vector(spec), 1.0, cfg, sk, F_RF=F)
    return steps, time.perf_counter() - t0


# CPU sample per config: steps per trial, so that one worker runs ~2-6 s
CPU_STEPS = {"C1": 50, "C2": 100, "C3": 40, "C4": 20, "C5": 8}


def cpu_rate(spec, eta, pool, steps, n_trials):
    """updates/s of the reference algorithm: n_trials trials x `steps` steps,
    one trial per worker process concurrently; total updates / busiest worker."""
    kw = dataclasses.asdict(spec)
    res = pool.map(_cpu_trial, [(kw, t, eta, steps) for t in range(n_trials)], chunksize=1)
    workers = pool._processes
    busy = [0.0] * workers
    for i, (_, sec) in enumerate(res):
        busy[i % workers] += sec
    return sum(r[0] for r in res) / max(busy)


def cpu_baseline(spec, eta, pool, cores):
    steps = min(spec.T, CPU_STEPS.get(spec.name, 20))
    n = cores
    v = cpu_rate(spec, eta, pool, steps, n)
    return {"value": v, "unit": "updates/s", "cores": cores, "kind": "port",
            "cpu_model": cpu_model(),
            "sample": f"{n} trials x first {steps} steps of {spec.name} {spec.dtype} "
                      f"({'conventional' if eta is None else f'eta={eta:g}'}), one trial per "
                      "worker process, oracle port of leorzf lowrank/precoding through the "
                      "_sweep_trial loop, BLAS 1 thread/worker, channel generation untimed"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    spec, eta = _spec(args)
    cores = _cores()
    steps = min(spec.T, CPU_STEPS.get(spec.name, 20))
    with _cpu_pool(cores, spec) as pool:
        for _ in range(args.warmup):
            cpu_rate(spec, eta, pool, 2, cores)
        wb = [cpu_rate(spec, eta, pool, steps, cores) for _ in range(args.steps)]
    v = statistics.median(wb)
    sample = (f"per step {cores} trials x first {steps} steps (one trial per worker), oracle "
              f"port of leorzf lowrank/precoding through the _sweep_trial loop, "
              f"{'F_RF = I_N verbatim' if spec.N <= 1024 else 'identity-elided F_RF (N = 4096)'}"
              f", BLAS 1 thread/worker; CPU {cpu_model()}")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "updates/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * cores * steps / v, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": spec.dtype,
        "data": "synthetic (SURVEY.md 8(d) seeded Rician drift channels)",
        "config": {"workload": workload_desc(spec, eta)},
        "cpu_baseline": {"value": v, "unit": "updates/s", "cores": cores, "kind": "port",
                         "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": v, "unit": "updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU leg

def _leo_cpu_job(job):
    """One LEO pass prefix of every method (oracle port of harness._sweep_trial
    with the reference's hybrid beams), timed inside the worker."""
    cfg_kw, trial, steps = job
    from oracle import leo as OL
    from paper_2512_16543_b200.leo import ScenarioConfig
    cfg = ScenarioConfig(**cfg_kw)
    etas = sorted(set(cfg.eta_list), reverse=True)
    specs = [(OL.label_of(None), None)] + [(OL.label_of(e), e) for e in etas]
    t0 = time.perf_counter()
    OL.sweep_trial(cfg, specs, trial, cfg.seed, steps=steps)
    return steps * len(specs), time.perf_counter() - t0


def leo_side(args, dev, world, max_over_ranks):
    """The reference's own default campaign (leorzf ScenarioConfig defaults: 50
    LEO passes x 2400 snapshots x 4 methods, hybrid DFT beams) through the
    run_campaign drop-in, timed on the device (max over ranks)."""
    import dataclasses
    import multiprocessing as mp
    import torch
    from paper_2512_16543_b200 import leo as L
    cfg = L.ScenarioConfig().validate()
    L.run_campaign(cfg.with_(mc_runs=2 * world, pass_s=10.0), device=dev)     # warm-up
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = L.run_campaign(cfg, device=dev)
    e1.record()
    torch.cuda.synchronize(dev)
    ms = max_over_ranks(e0.elapsed_time(e1))
    n_methods = len(res.labels)
    upd = cfg.mc_runs * cfg.n_snapshots * n_methods
    out = {"value": upd / (ms / 1e3), "unit": "updates/s", "ms": ms,
           "workload": f"leorzf default ScenarioConfig campaign: {cfg.mc_runs} passes x "
                       f"{cfg.n_snapshots} snapshots x {n_methods} methods (K = N_RF = 16, 16x16 "
                       "UPA, DFT beams), channels + beams + precoders + rates + reduction on "
                       "the device",
           "table": [[r.method_label, r.savings_pct, r.degradation_pct] for r in res.table.rows]}
    if world == 1 and not args.no_cpu:
        cores = _cores()
        kw = dataclasses.asdict(cfg)
        steps = 120
        saved = {k: os.environ.get(k) for k in _BLAS_ENV}
        for k in _BLAS_ENV:
            os.environ[k] = "1"
        try:
            with mp.get_context("spawn").Pool(cores, initializer=_cpu_init) as pool:
                pool.map(_leo_cpu_job, [(kw, 0, 2)] * cores)
                r = pool.map(_leo_cpu_job, [(kw, t, steps) for t in range(cores)], chunksize=1)
        finally:
            for k, v in saved.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        out["cpu_baseline"] = {"value": sum(u for u, _ in r) / max(sec for _, sec in r),
                               "unit": "updates/s", "cores": cores, "kind": "port",
                               "sample": f"{cores} passes x first {steps} snapshots x "
                                         f"{n_methods} methods, one pass per worker"}
    return out



class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.lines = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks(torch, dev):
    """FP64 / FP32 dense GEMM peaks measured now (cuBLAS via torch.matmul),
    since MEASURED_PEAKS.json only has HBM and bf16."""
    out = {}
    for name, dt in (("fp64", torch.float64), ("fp32", torch.float32), ("tf32", torch.float32)):
        n = 8192
        torch.backends.cuda.matmul.allow_tf32 = name == "tf32"
        a = torch.randn(n, n, dtype=dt, device=dev)
        b = torch.randn(n, n, dtype=dt, device=dev)
        for _ in range(2):
            a @ b
        best = 1e9
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            a @ b
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) / 1e3)
        out[name] = 2 * n ** 3 / best / 1e12
        del a, b
    torch.backends.cuda.matmul.allow_tf32 = False
    # 3xTF32 (hi*hi + hi*lo + lo*hi): three TF32 products per real product
    out["tf32x3_effective"] = out["tf32"] / 3.0
    return out


def ncu_traffic(kernel: str, spec, B: int, chunk: int):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of the
    dominant kernel from the committed ncu launch list of the same workload
    (profiles/r02_traffic_<config>_<dtype>.json, scripts/ncu_summary.py traffic),
    matched by kernel and grid size; (None, None) when not captured."""
    path = ROOT / "profiles" / f"r02_traffic_{spec.name}_{spec.dtype}.json"
    if not path.exists():
        return None, None
    tab = json.loads(path.read_text())
    K, N = spec.K, spec.N
    T = "double" if spec.dtype == "c128" else "float"
    items = B * chunk
    keys = {
        "dmma_hn_kernel:W": f"void lrz::zgemm_dmma_kernel<{T}, 0, 1, 0, 0, 0> grid"
                            f"({items * -(-N // 64) * -(-K // 64)},1,1)",
        "w_dmma_direct_kernel": f"void lrz::w_dmma_direct_kernel<{T}, 1> grid"
                                f"({items * -(-N // 32) * -(-(-(-K // 32)) // 4)},1,1)",
        "w_dmma_3m_tiled_kernel": f"void lrz::w_dmma_3m_tiled_kernel<{T}> grid"
                                  f"({items * -(-N // 64) * -(-K // 64)},1,1)",
        "gram_dmma_off_kernel": f"void lrz::gram_dmma_off_kernel<{T}> grid"
                                f"({-(-items * (K // 32) * (K // 32 - 1) // 2 // 4)},1,1)",
    }
    k = keys.get(kernel)
    if k is None or k not in tab:
        return None, None
    return tab[k]["dram_bytes_per_launch"], (
        f"ncu dram__bytes_read.sum + dram__bytes_write.sum per launch, {path.relative_to(ROOT)}")


def kernel_model(name: str, spec, items: int, D: int, Dtot: int, r_mean: float,
                 n_full: int, n_wb: int):
    """Algorithmic (flops, compulsory HBM bytes) of ONE launch of an
    instrumented kernel processing `items` (trial, step) items (SURVEY.md 8(d)
    'Algorithmic counts'; complex MAC = 8 flops, Hermitian outputs counted
    once; c = bytes per element of H; K x K matrices complex128)."""
    K, N = spec.K, spec.N
    c = 8 if spec.dtype == "c64" else 16
    nb = (K + 31) // 32
    if name in ("dmma_hn_kernel:W", "w_dmma_direct_kernel"):   # W = H^H A^-1 + ||W||^2
        return (8 * K * K * N + 8 * N * K) * items, (K * N * c + K * K * 16 + N * K * c) * items
    if name == "w_dmma_3m_tiled_kernel":
        # the 3M complex product executes three real products per complex one: 6 K^2 N
        # real flops for SURVEY 8(d)'s 8 K^2 N (bench reports both, see roofline_table)
        return (6 * K * K * N + 8 * N * K) * items, (K * N * c + K * K * 16 + N * K * c) * items
    if name == "coupling_dmma_3m_tiled":
        return 6 * K ** 3 * items, 3 * K * K * 16 * items
    if name == "tc_w_kernel":                      # W on tcgen05 (3xTF32, complex64)
        return (8 * K * K * N + 8 * N * K) * items, (K * N * c + N * K * c + 8 * (2 * K) ** 2) * items
    if name in ("dmma_hn_kernel:coupling", "coupling_dmma_direct"):   # (G - alpha I) A^-1, SURVEY A.6
        return 8 * K ** 3 * items, 3 * K * K * 16 * items
    if name == "precode_dmma32_kernel":            # W + norm + coupling + SINR fused
        # (executed flops: the W slabs run the 3M product, 6 K^2 N for SURVEY 8(d)'s 8 K^2 N)
        return ((6 * K * K * N + 8 * N * K + 8 * K ** 3 + 8 * K * K) * items,
                (K * N * c + N * K * c + 2 * K * K * 16) * items)
    if name == "gram_dmma_kernel":                 # diagonal 32-row blocks (lower incl. diag)
        kd = min(K, 32)
        return nb * 4 * kd * (kd + 1) * N * items, (K * N * c + K * K * 16) * items
    if name == "gram_dmma_off_kernel":             # K > 32: every lower 32 x 32 block
        # algorithmic Hermitian count 4 K (K + 1) N (executed: nb (nb + 1) / 2 full blocks)
        return 4 * K * (K + 1) * N * items, (K * N * c + K * K * 16) * items
    if name == "gram_dmma_3m_tiled_kernel":        # 3M product: 3 K (K + 1) N executed flops
        return 3 * K * (K + 1) * N * items, (K * N * c + K * K * 16) * items
    if name in ("dmma_hn_kernel:sketch_Y", "dmma_hn_kernel:sketch_W"):
        return 8 * K * K * Dtot * items, (K * K * 16 + 2 * K * Dtot * 16) * items
    if name == "sketch_dmma_kernel":               # Y = dA Omega and W = dA Y, K <= 32
        return 16 * K * K * Dtot * items, (K * K * 16 + 2 * K * Dtot * 8 + 2 * K * Dtot * 16) * items
    if name == "arsvd_screen_kernel":              # per iteration: Gram, Cholesky, X rows
        return 12 * K * Dtot * D * items, (2 * K * Dtot * 16 + K * K * 16) * items
    if name in ("chain_steps (all kernels)", "chain_kernel"):
        r = max(r_mean, 1.0)
        return ((24 * K * K * r + 16 * K * r * r + 8 * r ** 3 + 8 * K * K * r) * n_wb,
                (3 * K * K * 16 + 2 * K * r * 16) * n_wb)
    if name.startswith("herm_inverse") and name != "herm_inverse_kernel":
        # (herm_inverse_kernel only re-does the items the fast path flagged)
        return 4 * K ** 3 * n_full, 2 * K * K * 16 * n_full
    return None


def run_b200(args):
    import torch
    import torch.distributed as dist

    from paper_2512_16543_b200 import ops, scenario as S
    from paper_2512_16543_b200.omega import DeviceOmegaStreams
    from paper_2512_16543_b200.trajectory import TrajectoryConfig, TrajectoryRunner

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    spec, eta = _spec(args)
    B, T, K, Nn = spec.B, spec.T, spec.K, spec.N
    chunk = args.chunk or CHUNK.get(spec.name, T)
    trials = list(range(rank * B, (rank + 1) * B))
    tdt = torch.complex64 if spec.dtype == "c64" else torch.complex128
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def cfg_for(sp, e):
        return TrajectoryConfig(alpha=sp.alpha, eta=e, k_init=sp.k_init, p=sp.p, i_max=sp.i_max)

    # the back stages (the latency-bound chain first) get the higher stream
    # priority, so their small launches are scheduled ahead of the next chunk's
    # throughput-bound CTAs
    back = torch.cuda.Stream(dev, priority=-1)
    # "heavy" schedule: Grams and precoder products on a low-priority stream,
    # everything latency-bound on a high-priority one (run_chunk heavy_stream)
    heavy = torch.cuda.Stream(dev, priority=0)
    light = torch.cuda.Stream(dev, priority=-1)
    pipe_flags = torch.zeros(2, dtype=torch.int32, device=dev)

    def one_pass(sp, e, Hs, streams, noise, ch, prof=None, on_chunk=None, pipelined=False):
        """One pass of the hot path over B trials x T steps (T in chunks of ch):
        fresh runner, sketch windows regenerated on the device from the stream
        start, results of the last chunk returned.  Hs: list of per-chunk
        device channel tensors, or a callable (t0, t1) -> tensor.
        pipelined = True / "back": the runner's back stages (dispatcher,
        inversions, chain, precoder, rate) of chunk c run on a second stream
        while the front stages (Grams, arSVD) of chunk c + 1 proceed (run_chunk
        back_stream, sync=False: verifier flags accumulate in pipe_flags and are
        checked by the caller); at most two chunks in flight.
        pipelined = "heavy": the Grams of chunk c + 1 and the precoder products
        of chunk c back to back on a low-priority stream, the latency-bound
        stages between them on a high-priority one (run_chunk heavy_stream)."""
        b = noise.shape[0]
        rn = TrajectoryRunner(b, sp.K, sp.N, tdt if sp is spec else
                              (torch.complex64 if sp.dtype == "c64" else torch.complex128),
                              cfg_for(sp, e), dev)
        rn.prof = prof
        if e is not None:
            streams.raw.zero_()
            streams.consumed_total.zero_()
        outs, evs = [], []
        bounds = [(t0, min(sp.T, t0 + ch)) for t0 in range(0, sp.T, ch)]
        if pipelined == "heavy":
            get = lambda i: Hs[i] if isinstance(Hs, list) else Hs(*bounds[i])  # noqa: E731
            light.wait_stream(stream)
            with torch.cuda.stream(light):
                H_next = get(0)
                g_next = rn.gram_async(H_next, heavy)
                for i, (t0, t1) in enumerate(bounds):
                    H, g = H_next, g_next
                    if i + 1 < len(bounds):
                        # issued before this chunk's precoder: G(c+1) | W(c) on `heavy`
                        H_next = get(i + 1)
                        g_next = rn.gram_async(H_next, heavy)
                    else:
                        H_next = g_next = None
                    om = None if e is None else \
                        streams.window((t1 - t0) * rn.normals_per_step_max())
                    r = rn.run_chunk(H, noise, om, sync=False, heavy_stream=heavy, gram=g)
                    if r.flags is not None:
                        pipe_flags.add_(r.flags)
                    if e is not None:
                        streams.advance(r.consumed)
                    outs.append(r)
                    del H, g
            stream.wait_stream(light)
            stream.wait_stream(heavy)
            return outs
        for i, (t0, t1) in enumerate(bounds):
            if pipelined and i >= 2:
                stream.wait_event(evs[i - 2])     # back stages of chunk i - 2 done
            H = Hs[i] if isinstance(Hs, list) else Hs(t0, t1)
            if on_chunk is not None:
                on_chunk(i, "start")
            om = None if e is None else streams.window((t1 - t0) * rn.normals_per_step_max())
            if pipelined:
                r = rn.run_chunk(H, noise, om, sync=False, back_stream=back)
                if r.flags is not None:
                    pipe_flags.add_(r.flags)
                ev = torch.cuda.Event()
                ev.record(back)
                evs.append(ev)
            else:
                r = rn.run_chunk(H, noise, om)
            if e is not None:
                streams.advance(r.consumed)
            if on_chunk is not None:
                on_chunk(i, "end")
            outs.append(r)
        if pipelined:
            stream.wait_stream(back)
        return outs

    def pick_pipeline(sp, e, Hs, streams, noise, ch, ref, modes):
        """The fastest schedule among `modes` that reproduces the synchronous
        pass `ref` (verifier flags zero, same decisions and rates); False when
        none does.  Each candidate: one checked pass, then one timed pass."""
        best, best_ms, tried = False, None, {}
        for mode in modes:
            ops._WS.clear()
            torch.cuda.empty_cache()
            pipe_flags.zero_()
            tri = one_pass(sp, e, Hs, streams, noise, ch, pipelined=mode)
            torch.cuda.synchronize(dev)
            ok = int(pipe_flags.abs().sum().item()) == 0 and all(
                torch.equal(a.method, b_.method) and torch.equal(a.k_est, b_.k_est) and
                torch.equal(a.rates, b_.rates) for a, b_ in zip(ref, tri))
            del tri
            if not ok:
                tried[str(mode)] = None
                continue
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            one_pass(sp, e, Hs, streams, noise, ch, pipelined=mode)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            tried[str(mode)] = e0.elapsed_time(e1)
            # (the first candidate is kept unless a later one is more than 3 % faster:
            # one pass each is a noisy comparison)
            if best_ms is None or tried[str(mode)] < 0.97 * best_ms:
                best, best_ms = mode, tried[str(mode)]
        if len(modes) > 1:
            ops._WS.clear()      # per-stream scratch of the schedules not kept
            torch.cuda.empty_cache()
        return best, tried

    def summarize(outs):
        method = torch.cat([o.method for o in outs], 1).cpu().numpy()
        k_est = torch.cat([o.k_est for o in outs], 1).cpu().numpy()
        iters = torch.cat([o.iters for o in outs], 1).cpu().numpy()
        rates = torch.cat([o.rates for o in outs], 1).cpu().numpy()
        info = torch.cat([o.info for o in outs], 1).cpu().numpy()
        wb = int((method == 1).sum())
        return {"method_counts": {"full": int((method == 0).sum()), "woodbury": wb,
                                  "none": int((method == 2).sum())},
                "k_mean_woodbury": float(k_est[method == 1].mean()) if wb else 0.0,
                "iters_hist": {int(i): int(c) for i, c in zip(*np.unique(iters[iters > 0],
                                                                         return_counts=True))},
                "mean_sum_rate": float(rates.mean()), "finite": bool(np.isfinite(rates).all()),
                "singular_steps": int((info == 1).sum()), "_wb": wb,
                "_r": float(k_est[method == 1].mean()) if wb else 0.0,
                "_full": int((method == 0).sum())}

    def timed(fn, steps):
        barrier()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        last = None
        for _ in range(steps):
            last = fn()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        return max_over_ranks(e0.elapsed_time(e1)) / steps, last

    peaks = measured_peaks(torch, dev)
    mp_path = ROOT / "MEASURED_PEAKS.json"
    hbm = json.loads(mp_path.read_text())["hbm_gbs"] if mp_path.exists() else 6650.0

    def roofline_table(kprof, sp, steps, items_per_pass, summ, Dtot, D):
        """Per-kernel achieved vs roofline from CUDA-event times over the timed
        region: a kernel's algorithmic work over one pass (items_per_pass
        (trial, step) items; Woodbury / full-step counts for the chain and the
        inversions) divided evenly over its launches in the pass; the dominant
        kernel (largest total time) first."""
        rows = {}
        for name, (ms, n) in kprof.items():
            # FP64 pipe (DMMA / DFMA) for everything but the tcgen05 precoder, whose
            # 3xTF32 split runs three TF32 products per real product
            fpk = peaks["tf32x3_effective"] if name == "tc_w_kernel" else peaks["fp64"]
            if n == 0 or ms <= 0:
                continue
            per_launch = ms / n
            per_pass = n / max(steps, 1)
            m = kernel_model(name, sp, items_per_pass, D, Dtot, summ["_r"], summ["_full"],
                             summ["_wb"])
            if m is not None:
                m = (m[0] / per_pass, m[1] / per_pass)
            row = {"ms_total_per_step": ms / steps, "launches_per_step": n / steps,
                   "ms_per_launch": per_launch}
            if m is not None:
                f, b_ = m
                t = per_launch / 1e3
                t_f, t_b = f / (fpk * 1e12), b_ / (hbm * 1e9)
                if t_f >= t_b:
                    row.update(bound="tensor", achieved=f / t / 1e12, peak=fpk, unit="TFLOP/s")
                else:
                    row.update(bound="hbm", achieved=b_ / t / 1e9, peak=hbm, unit="GB/s")
                row["frac"] = row["achieved"] / row["peak"]
                row["flops_per_launch"] = f
                row["bytes_per_launch"] = b_
                if "3m_tiled" in name or name == "precode_dmma32_kernel":
                    # against SURVEY 8(d)'s four-product count (complex MAC = 8 flops)
                    extra = {"w_dmma_3m_tiled_kernel": 2 * sp.K * sp.K * sp.N,
                             "precode_dmma32_kernel": 2 * sp.K * sp.K * sp.N,
                             "coupling_dmma_3m_tiled": 2 * sp.K ** 3,
                             "gram_dmma_3m_tiled_kernel": sp.K * (sp.K + 1) * sp.N}[name]
                    f4 = f + extra * items_per_pass / per_pass
                    row["four_product_equivalent"] = {
                        "flops_per_launch": f4, "achieved": f4 / t / 1e12,
                        "frac": f4 / t / 1e12 / fpk,
                        "note": "3M complex product: 3 real DMMA products per complex one; "
                                "`achieved` counts the executed flops, this entry SURVEY "
                                "8(d)'s count (complex MAC = 8 flops)"}
            rows[name] = row
        return dict(sorted(rows.items(), key=lambda kv: -kv[1]["ms_total_per_step"]))

    def dominant(rows):
        for name, r in rows.items():
            if "frac" in r:
                out = {k: r[k] for k in ("bound", "achieved", "peak", "unit", "frac")}
                if "four_product_equivalent" in r:
                    out["four_product_equivalent"] = r["four_product_equivalent"]
                out.update(kernel=name, ms_per_launch=r["ms_per_launch"],
                           launches_per_step=r["launches_per_step"],
                           algorithmic={"flops_per_launch": r["flops_per_launch"],
                                        "bytes_per_launch": r["bytes_per_launch"]},
                           peak_source=(("measured now: cuBLAS TF32 GEMM 8192^3 / 3 (3xTF32 "
                                         "split), MEASURED_PEAKS.json has no TF32 entry")
                                        if name == "tc_w_kernel" else
                                        ("measured now: cuBLAS DGEMM 8192^3 via torch.matmul "
                                         "(MEASURED_PEAKS.json has no FP64 entry)"))
                           if r["unit"] == "TFLOP/s" else "MEASURED_PEAKS.json hbm_gbs",
                           traffic=None)
                return out
        return None

    def sketch_dims(sp):
        ds, k0 = [], sp.k_init
        for _ in range(sp.i_max):
            ds.append(min(k0 + sp.p, sp.K))
            k0 *= 2
        return sum(ds), max(ds)

    # ================================================================ headline
    noise = torch.full((B, K), spec.noise_var, dtype=torch.float64, device=dev)
    chans = S.DeviceChannels(spec, trials, dev)
    # inputs resident in HBM before timing (device synthesis = the host generator's
    # channels, tests/test_gpu_rng.py); one tensor per T-chunk so each is contiguous
    H_chunks = [chans.generate(t0, min(T, t0 + chunk)) for t0 in range(0, T, chunk)]
    torch.cuda.synchronize(dev)
    h_bytes = sum(h.numel() * h.element_size() for h in H_chunks)
    streams = DeviceOmegaStreams.for_method(spec.seed, eta, trials, dev)
    # cross-chunk pipelining (run_chunk back_stream) when one speculative arSVD
    # pass settles every chunk -- checked on a warm-up pass (verifier flags zero
    # and the same results as the synchronous pass)
    ref_sync = one_pass(spec, eta, H_chunks, streams, noise, chunk)
    torch.cuda.synchronize(dev)
    pipelined, pipe_tried = pick_pipeline(spec, eta, H_chunks, streams, noise, chunk, ref_sync,
                                          PIPE_MODES[args.pipe])
    del ref_sync
    wb = lambda: one_pass(spec, eta, H_chunks, streams, noise, chunk,  # noqa: E731
                          pipelined=pipelined)
    full = lambda: one_pass(spec, None, H_chunks, None, noise, chunk,  # noqa: E731
                            pipelined=pipelined)
    for _ in range(args.warmup):
        wb()
        full()
    torch.cuda.synchronize(dev)
    l0 = ops.LAUNCHES[0]
    ref_outs = wb()
    launches = ops.LAUNCHES[0] - l0
    summ = summarize(ref_outs)
    l0 = ops.LAUNCHES[0]
    full()
    launches_full = ops.LAUNCHES[0] - l0
    with Clocks(local) as clk:
        ops.prof_enable(True, dev)
        ms_wb, outs = timed(wb, args.steps)
        kprof = ops.prof_collect(dev)
        ops.prof_enable(False, dev)
        ms_full, _ = timed(full, args.steps)
    summ_t = summarize(outs)
    if summ_t["method_counts"] != summ["method_counts"]:
        raise RuntimeError("timed passes differ from the reference pass")
    if pipelined and int(pipe_flags.abs().sum().item()):
        raise RuntimeError("pipelined passes left unverified arSVD steps")
    updates = B * T
    value = world * updates / (ms_wb / 1e3)
    value_full = world * updates / (ms_full / 1e3)
    Dtot, D = sketch_dims(spec)
    ktab = roofline_table(kprof, spec, args.steps, B * T, summ, Dtot, D)
    roof = dominant(ktab)
    if roof is not None:
        roof["traffic"], roof["traffic_source"] = ncu_traffic(roof["kernel"], spec, B, chunk)
    # stage split: one more pass with events between the runner's stages; when the
    # timed passes overlap two streams, the per-kernel table is taken from this
    # unpipelined pass too (a kernel's event time then excludes the other stream's
    # kernels it shared the SMs with); the dominant kernel's `roofline` stays the
    # timed region's measurement
    prof = []
    if pipelined:
        # the pipelined passes' large buffers belong to the back stream's allocator
        # pool: release them and warm the front stream's pool with one untimed pass,
        # so the stage events below do not bracket cudaMalloc / cudaFree stalls
        torch.cuda.synchronize(dev)
        ops._WS.clear()
        torch.cuda.empty_cache()
        one_pass(spec, eta, H_chunks, streams, noise, chunk)
        torch.cuda.synchronize(dev)
        ops.prof_enable(True, dev)
    one_pass(spec, eta, H_chunks, streams, noise, chunk, prof=prof)
    torch.cuda.synchronize(dev)
    if pipelined:
        ktab = roofline_table(ops.prof_collect(dev), spec, 1, B * T, summ, Dtot, D)
        ops.prof_enable(False, dev)
    stages = {}
    for name, a, b_ in prof:
        stages[name] = stages.get(name, 0.0) + a.elapsed_time(b_)
    del H_chunks
    ops._WS.clear()
    torch.cuda.empty_cache()

    # ================================================================ e2e
    e2e = None
    if not args.no_e2e:
        be = min(args.e2e_trials, B)
        ch_e = chunk
        ech = S.DeviceChannels(spec, trials[:be], dev)
        n_chunks = (T + ch_e - 1) // ch_e
        host = []
        for i in range(n_chunks):     # pinned host channels (the caller's inputs)
            t0, t1 = i * ch_e, min(T, (i + 1) * ch_e)
            hd = ech.generate(t0, t1)
            hp = torch.empty(hd.shape, dtype=hd.dtype).pin_memory()
            hp.copy_(hd)
            host.append(hp)
            del hd
        bufs = [torch.empty(host[0].shape, dtype=tdt, device=dev) for _ in range(2)]
        noise_e = noise[:be].contiguous()
        st_e = DeviceOmegaStreams.for_method(spec.seed, eta, trials[:be], dev)
        copy_s = torch.cuda.Stream(dev)
        out_pin = {}
        d2h = [0]

        def e2e_pass():
            rn = TrajectoryRunner(be, K, Nn, tdt, cfg_for(spec, eta), dev)
            st_e.raw.zero_()
            st_e.consumed_total.zero_()
            ready = []

            def enqueue(i):
                buf = bufs[i % 2]
                if buf.shape[1] != host[i].shape[1]:
                    buf = bufs[i % 2] = torch.empty(host[i].shape, dtype=tdt, device=dev)
                with torch.cuda.stream(copy_s):
                    copy_s.wait_stream(stream)      # the buffer's previous reader is done
                    buf.copy_(host[i], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(copy_s)
                ready.append(ev)

            enqueue(0)
            nbytes = 0
            for i in range(n_chunks):
                if i + 1 < n_chunks:
                    enqueue(i + 1)
                stream.wait_event(ready[i])
                t1 = min(T, (i + 1) * ch_e)
                om = st_e.window((t1 - i * ch_e) * rn.normals_per_step_max())
                r = rn.run_chunk(bufs[i % 2], noise_e, om)
                st_e.advance(r.consumed)
                for nm in ("rates", "per_ut", "method", "k_est"):
                    t_ = getattr(r, nm)
                    key = (nm, i)
                    if key not in out_pin or out_pin[key].shape != t_.shape:
                        out_pin[key] = torch.empty(t_.shape, dtype=t_.dtype).pin_memory()
                    out_pin[key].copy_(t_, non_blocking=True)
                    nbytes += t_.numel() * t_.element_size()
            d2h[0] = nbytes

        e2e_pass()
        ms_e2e, _ = timed(e2e_pass, max(2, min(args.steps, 3)))
        e2e = {"value": world * be * T / (ms_e2e / 1e3), "unit": "updates/s",
               "h2d_bytes_per_step": int(sum(h.numel() * h.element_size() for h in host)),
               "d2h_bytes_per_step": int(d2h[0]), "ms_per_step": ms_e2e,
               "trials_per_gpu": be,
               "path": "TrajectoryRunner.run_chunk (public batched API over the C ABI) on "
                       f"{be} of the {B} trials x all {T} steps: each {ch_e}-step chunk of "
                       "pinned host channels copied H2D on a copy stream (double-buffered, "
                       "overlapping the previous chunk's compute), sketch normals from the "
                       "harness's PCG64 streams on the device, rates / per-UT rates / methods / "
                       "ranks copied back to pinned host memory"}
        del host, bufs
        torch.cuda.empty_cache()

    # ================================================================ per-config keys
    configs = {}
    if not args.no_extra:
        cores = _cores()
        runs = [
            ("C1_c128", "C1", {}, [spec_eta_default, None], 2),
            ("C2_c128", "C2", {}, [spec_eta_default, None], 5),
            ("C2_c128_eta0.9", "C2", {}, [0.9], 5),      # chunk 100: cross-chunk pipelining
            ("C2_c64", "C2", {"dtype": "c64"}, [spec_eta_default, None], 5),
            ("C3_c64", "C3", {}, [spec_eta_default, None], 1),
            ("C5_c64", "C5", {"dtype": "c64"}, [spec_eta_default, None], 1),
        ]
        for cap in (4, 8, 16, 32):
            for tol in (1e-2, 1e-3, 1e-4):
                lab = f"C4_cap{cap}_tol{tol:g}"
                runs.append((lab, "C4", {"cap": cap, "tol": tol},
                             [spec_eta_default] + ([None] if (cap, tol) == (16, 1e-3) else []),
                             1))
        for lab, name, ov, etas, reps in runs:
            sp = S.CONFIGS[name].with_(**ov)
            # the next chunk's Grams / screen rounds overlap this chunk's chain
            ch_over = 100 if lab == "C2_c128_eta0.9" else None
            if args.quick:
                sp = sp.with_(T=min(sp.T, 2 * CHUNK[name]))
            configs[lab] = run_config(sp, etas, reps, rank, world, dev, one_pass, summarize,
                                      roofline_table, dominant, sketch_dims, timed, ops, S,
                                      DeviceOmegaStreams, torch, pipe_flags, ch_over,
                                      pick_pipeline, PIPE_MODES[args.pipe])
            ops._WS.clear()          # grow-only scratch of this config's shapes
            torch.cuda.empty_cache()
        if rank == 0 and world == 1 and not args.no_cpu:
            for lab, name, ov, etas, _ in runs:
                if lab.startswith("C4") and lab != "C4_cap16_tol0.001":
                    continue
                sp = S.CONFIGS[name].with_(**ov)
                e = etas[0] if etas[0] is not None else sp.eta
                e = sp.eta if e == "default" else e
                with _cpu_pool(cores, sp) as pool:
                    configs[lab]["cpu_baseline"] = cpu_baseline(sp, e, pool, cores)

    leo = None
    if not args.no_extra:
        ops._WS.clear()
        torch.cuda.empty_cache()
        leo = leo_side(args, dev, world, max_over_ranks)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cores = _cores()
        with _cpu_pool(cores, spec) as pool:
            cpu = cpu_baseline(spec, eta, pool, cores)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "updates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_wb,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": spec.dtype,
            "data": "synthetic (SURVEY.md 8(d) seeded Rician drift channels, synthesised on the "
                    "device = the host generator's values; the reference has no public dataset)",
            "config": {"workload": workload_desc(spec, eta)},
            "l2": "inputs larger than L2 (H = %.1f GB per GPU resident in HBM), no flush needed"
                  % (h_bytes / 1e9),
            "updates_per_step": updates * world,
            "method": "WB-arSVD (eta = 1 - tol, SURVEY D3), every step after the first a "
                      "Woodbury update; Omega generated on the device inside every step; W "
                      "written to HBM",
            "pipelined": pipelined,
            "pipeline_candidates_ms": pipe_tried,
            "full_inverse": {"value": value_full, "unit": "updates/s", "ms_per_step": ms_full,
                             "gpu_launches": launches_full},
            "roofline": roof,
            "kernels": ktab,
            "kernels_timing": ("CUDA events per launch, one unpipelined pass (the timed passes "
                               "overlap two streams); `roofline` is the timed region's") if pipelined
                              else "CUDA events per launch over the timed passes",
            "stages_ms_per_step": stages,
            "peaks_measured": peaks,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            **{k: v for k, v in summ.items() if not k.startswith("_")},
            "configs": configs,
        }
        if leo:
            line["leo_campaign"] = leo
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


spec_eta_default = "default"
# stream schedules tried per config (bench picks the fastest that reproduces the
# synchronous pass): "heavy" = run_chunk heavy_stream, "back" = run_chunk back_stream
PIPE_MODES = {"auto": ("back", "heavy"), "heavy": ("heavy",), "back": ("back",), "off": ()}
# default "back": the heavy schedule measured +1.5 % at C5 c128 (800 vs 812 ms per
# pass) and within +-3 % elsewhere, while the precoder kernel's event time then
# includes the latency-bound kernels its CTAs share the SMs with


def run_config(sp, etas, reps, rank, world, dev, one_pass, summarize, roofline_table, dominant,
               sketch_dims, timed, ops, S, DeviceOmegaStreams, torch, pipe_flags, chunk=None,
               pick_pipeline=None, pipe_modes=()):
    """One BASELINE config at its full trial count and T; each method timed over
    `reps` passes after one warm-up pass.  The channels of the whole pass are
    resident in HBM before the timed region when they fit (every config but
    C4): `updates_per_s` is then the pass itself.  C4's 215 GB pass is
    streamed -- every T-chunk synthesised on the device inside the timed pass --
    so its `updates_per_s` includes the channel synthesis (`channels`:
    "streamed"; the synthesis timed alone is reported beside it)."""
    B, T = sp.B, sp.T
    trials = list(range(rank * B, (rank + 1) * B))
    ch = min(T, chunk or CHUNK.get(sp.name, T))
    chans = S.DeviceChannels(sp, trials, dev)
    noise = torch.full((B, sp.K), sp.noise_var, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    h_chunk = B * ch * sp.K * sp.N * (8 if sp.dtype == "c64" else 16)
    n_ch = (T + ch - 1) // ch
    resident = n_ch * h_chunk <= 0.45 * torch.cuda.get_device_properties(dev).total_memory
    out = {"workload": None, "B": B, "T": T, "chunk": ch, "dtype": sp.dtype,
           "channels": "resident" if resident else "streamed"}
    if resident:
        Hsrc = [chans.generate(t0, min(T, t0 + ch)) for t0 in range(0, T, ch)]
        torch.cuda.synchronize(dev)
    else:
        Hsrc = chans.generate
        # the synthesis of one pass's channels timed alone (context for `updates_per_s`)
        chans.generate(0, ch)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        e0.record(stream)
        for t0 in range(0, T, ch):
            chans.generate(t0, min(T, t0 + ch))
        e1.record(stream)
        torch.cuda.synchronize(dev)
        out["channels_ms_per_pass_alone"] = e0.elapsed_time(e1)
    for e in etas:
        e = sp.eta if e == "default" else e
        streams = None if e is None else DeviceOmegaStreams.for_method(sp.seed, e, trials, dev)
        evs = []

        def mark(i, what):
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(stream)
            evs.append(ev)

        # cross-chunk pipelining when a warm-up pass shows it reproduces the
        # synchronous pass (verifier flags zero, same decisions and rates)
        torch.cuda.reset_peak_memory_stats(dev)
        ref = one_pass(sp, e, Hsrc, streams, noise, ch)
        torch.cuda.synchronize(dev)
        modes = list(pipe_modes)
        if not resident and torch.cuda.max_memory_allocated(dev) + 3 * h_chunk > \
                0.8 * torch.cuda.get_device_properties(dev).total_memory:
            # the heavy schedule keeps one more channel chunk (and its Grams) alive
            modes = [m for m in modes if m != "heavy"]
        pipelined, tried = pick_pipeline(sp, e, Hsrc, streams, noise, ch, ref, modes)
        del ref
        if pipelined:
            torch.cuda.synchronize(dev)
        run = lambda: one_pass(sp, e, Hsrc, streams, noise, ch,  # noqa: E731
                               on_chunk=None if pipelined else mark, pipelined=pipelined)
        # warm-up: two passes for the short ones (the caching allocator settles its
        # cross-stream reuse only on the second pipelined pass)
        run()
        if min((v for v in tried.values() if v), default=1e9) < 500.0:
            run()
        torch.cuda.synchronize(dev)
        evs.clear()
        ops.prof_enable(True, dev)
        ms, outs = timed(run, reps)
        kprof = ops.prof_collect(dev)
        ops.prof_enable(False, dev)
        if pipelined or resident:
            # resident channels: the pass is the runner; streamed (C4): the pass
            # includes the synthesis (under two overlapping streams there is no
            # runner-only time to separate out)
            runner_ms = ms
        else:
            runner_ms = sum(evs[i].elapsed_time(evs[i + 1])
                            for i in range(0, len(evs), 2)) / reps
        summ = summarize(outs)
        Dtot, D = sketch_dims(sp)
        kreps = reps
        if pipelined:
            # per-kernel rooflines from one more, unpipelined pass: under the two
            # overlapping streams of the timed passes a kernel's event time includes
            # the other stream's kernels it shares the SMs with
            torch.cuda.synchronize(dev)
            ops.prof_enable(True, dev)
            one_pass(sp, e, Hsrc, streams, noise, ch)
            torch.cuda.synchronize(dev)
            kprof = ops.prof_collect(dev)
            ops.prof_enable(False, dev)
            kreps = 1
        ktab = roofline_table(kprof, sp, kreps, B * T, summ, Dtot, D)
        key = "conventional" if e is None else f"wb_eta{e:g}"
        out[key] = {
            "updates_per_s": world * B * T / (runner_ms / 1e3),
            "ms_per_pass": runner_ms, "pipelined": pipelined,
            "pipeline_candidates_ms": tried, "roofline": dominant(ktab),
            "kernel_timing": ("CUDA events per launch, unpipelined pass (the timed passes "
                              "overlap two streams)") if pipelined else
                             "CUDA events per launch over the timed passes",
            "kernels_top": dict(list(ktab.items())[:6]),
            **{k: v for k, v in summ.items() if not k.startswith("_")}}
        out["workload"] = workload_desc(sp, e if e is not None else sp.eta)
    return out



def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
