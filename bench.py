#!/usr/bin/env python
"""RZF precoder updates/s (WB-arSVD vs full inverse) on one B200 -- BASELINE.json metric.

Workload (BASELINE.json configs[1], SURVEY.md 8(d) "C2"): N = 256 (16x16 UPA),
K = 32 users, T = 200 orbit steps, B = 64 Monte-Carlo trials per GPU, SNR
10 dB (alpha = K/SNR), arSVD tolerance 1e-3 (eta = 0.999), rank cap 16
(i_max = 4), oversampling p = 5, complex128.  One bench "step" = one pass
of the hot path over the whole batch: B * T = 12,800 precoder updates, each
producing A^-1_t, W_t and the sum-rate (harness._sweep_trial semantics).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

--impl reference times the reference algorithm on the host CPU (the numpy
oracle port in oracle/, all cores, BLAS pinned to one thread per worker like
harness.py:284-293).  Multi-GPU: torchrun, one rank per GPU, trials sharded
by rank (weak scaling, no data-path collective), max-over-ranks timing.
"""

from __future__ import annotations

import argparse
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--dtype", default="c128", choices=["c128", "c64"])
    ap.add_argument("--snr", type=float, default=10.0)
    ap.add_argument("--eta", type=float, default=None)
    ap.add_argument("--trials", type=int, default=None, help="trials per GPU (default: config B)")
    ap.add_argument("--T", type=int, default=None)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the c64 side measurement")
    ap.add_argument("--no-graph", action="store_true",
                    help="launch every step eagerly instead of replaying its CUDA graph")
    return ap.parse_args()


def _spec(args):
    from paper_2512_16543_b200 import scenario as S
    spec = S.CONFIGS[args.config].with_(dtype=args.dtype, snr_db=args.snr)
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
        kw["T"] = 3
        _cpu_trial((kw, 0, 1.0 - kw["tol"]))
        _cpu_trial((kw, 0, None))


def _cpu_pool(cores, spec):
    """Spawned worker pool with BLAS pinned to one thread per process."""
    import dataclasses
    import multiprocessing as mp
    saved = {k: os.environ.get(k) for k in _BLAS_ENV}
    for k in _BLAS_ENV:
        os.environ[k] = "1"
    try:
        return mp.get_context("spawn").Pool(cores, initializer=_cpu_init,
                                            initargs=(dataclasses.asdict(spec),))
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _cpu_trial(job):
    """One trial of the reference algorithm (oracle port) on one core; channel
    generation is outside the timed region, F_RF = I_N verbatim."""
    spec_kw, trial, eta = job
    from oracle import port, sweep
    from paper_2512_16543_b200 import scenario as S
    spec = S.ScenarioSpec(**spec_kw)
    H = S.trial_channels(spec, trial)
    if spec.dtype == "c64":
        H = H.astype(np.complex64)
    F = np.eye(spec.N)
    cfg = None if eta is None else port.Cfg(eta, spec.k_init, spec.p, spec.i_max)
    sk = None if eta is None else np.random.default_rng(
        S.stream_seed(spec.seed, S.method_label(eta), trial))
    t0 = time.perf_counter()
    sweep.sweep_trial(H, spec.alpha, S.noise_vector(spec), 1.0, cfg, sk, F_RF=F)
    return spec.T, time.perf_counter() - t0


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


def _cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_rate(spec, eta, n_trials, pool):
    """updates/s of the reference algorithm over n_trials trials run one per
    worker process concurrently: total updates / busiest worker's time."""
    import dataclasses
    kw = dataclasses.asdict(spec)
    jobs = [(kw, t, eta) for t in range(n_trials)]
    res = pool.map(_cpu_trial, jobs, chunksize=1)
    workers = pool._processes
    busy = [0.0] * workers
    for i, (_, sec) in enumerate(res):
        busy[i % workers] += sec
    return sum(r[0] for r in res) / max(busy)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    spec, eta = _spec(args)
    cores = _cores()
    n_trials = min(spec.B, cores)
    with _cpu_pool(cores, spec) as pool:
        for _ in range(args.warmup):
            cpu_rate(spec.with_(T=min(spec.T, 20)), eta, min(n_trials, cores), pool)
        wb = [cpu_rate(spec, eta, n_trials, pool) for _ in range(args.steps)]
        full = [cpu_rate(spec, None, n_trials, pool) for _ in range(max(1, args.steps // 2))]
    v = statistics.median(wb)
    sample = (f"{n_trials} trials x {spec.T} steps per step (one trial per worker), oracle port "
              f"of leorzf lowrank/precoding with F_RF = I_N verbatim, BLAS 1 thread/worker")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "updates/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * n_trials * spec.T / v, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": spec.dtype,
        "data": "synthetic (SURVEY.md 8(d) seeded Rician drift channels)",
        "config": {"workload": workload_desc(spec, eta)},
        "full_inverse": {"value": statistics.median(full), "unit": "updates/s"},
        "cpu_baseline": {"value": v, "unit": "updates/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": v, "unit": "updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU leg

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
    for name, dt in (("fp64", torch.float64), ("fp32", torch.float32)):
        n = 8192 if name == "fp64" else 8192
        torch.backends.cuda.matmul.allow_tf32 = False
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
    return out


def stage_model(spec, T, B, k_mean, iters_hist, wb_steps):
    """Algorithmic flops / compulsory HBM bytes per stage for one bench step
    (SURVEY.md 8(d) 'Algorithmic counts'; c = bytes per complex element of H;
    K x K matrices are complex128 = 16 B)."""
    K, N = spec.K, spec.N
    c = 8 if spec.dtype == "c64" else 16
    BT = B * T
    n_sk = B * (T - 1)
    m = {}
    m["gram"] = (4 * K * (K + 1) * N * BT, (K * N * c + K * K * 16) * BT)
    # difference form G_t - G_{t-1} of the fp64 Grams (TrajectoryConfig.delta "auto":
    # the DMMA Grams accumulate in fp64 for both dtypes)
    # (each Gram is read once as G_t and once as G_{t-1}: compulsory = one read + dA out)
    m["gram_delta"] = (2 * K * K * n_sk, 2 * K * K * 16 * n_sk)
    widths = []
    k0 = spec.k_init
    for _ in range(spec.i_max):
        widths.append(min(k0 + spec.p, K))
        k0 *= 2
    f_ar = 0.0
    b_ar = 0.0
    for it, cnt in iters_hist.items():
        ds = widths[:it]
        f_ar += cnt * (4 * K * K + sum(16 * K * K * d + 32 * K * d * d for d in ds))
        b_ar += cnt * sum(K * K * 16 + 2 * K * d * 8 for d in ds)
    m["arsvd"] = (f_ar, b_ar)
    n_full = BT - wb_steps
    m["inverse"] = ((4 / 3 + 8 / 3) * K ** 3 * n_full, 2 * K * K * 16 * n_full)
    r = max(k_mean, 1.0)
    m["chain"] = ((24 * K * K * r + 16 * K * r * r + 8 * r ** 3 + 8 * K * K * r) * wb_steps,
                  (2 * K * K * 16 + 2 * K * r * 16) * wb_steps)
    # W = H^H A^-1, ||W||_F^2, H W from the Gram shortcut (G - alpha I) A^-1 (K^3,
    # the flops actually executed, not the 8 K^2 N product it replaces), SINR
    m["precode_rate"] = ((8 * K * K * N + 8 * N * K + 8 * K ** 3 + 8 * K * K) * BT,
                         (K * N * c + N * K * c + 2 * K * K * 16) * BT)
    return m


# kernels (name fragment, launches per WB step) behind each bench stage
STAGE_KERNELS = {
    "arsvd": [("sketch_dmma_kernel", 1), ("arsvd_screen_kernel", 1), ("arsvd_kernel", 1)],
    "gram": [("gram_dmma_kernel", 1)],
    "precode_rate": [("precode_dmma32_kernel", 1)],
    "inverse": [("herm_inverse_warp_kernel", 1), ("herm_inverse_kernel", 1)],
    "omega_rng": [("rng_pass_a", 1), ("rng_pass_b", 1), ("rng_pass_c", 1)],
}


# kernels that carry a stage's work (for picking the dominant kernel)
STAGE_MAIN_KERNELS = {"arsvd": 2, "omega_rng": 3}


def stage_traffic(stage, spec):
    """DRAM bytes per step of a stage (sum over its kernels, per launch x launches)
    from the committed ncu capture of the same command (profiles/, C2 c128 only)."""
    path = ROOT / "profiles" / "r01_traffic_C2_c128.json"
    if spec.name != "C2" or spec.dtype != "c128" or not path.exists() or stage not in STAGE_KERNELS:
        return None
    tab = json.loads(path.read_text())
    tot = 0.0
    for frag, n in STAGE_KERNELS[stage]:
        hits = [v for k, v in tab.items() if k.split("<")[0].endswith(frag)]
        if not hits:
            return None
        tot += hits[0]["dram_bytes_per_launch"] * n
    return {"bytes_per_step": tot, "source": f"ncu dram__bytes_read.sum + dram__bytes_write.sum, "
                                               f"{path.relative_to(ROOT)}"}


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
    trials = list(range(rank * B, (rank + 1) * B))

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- inputs (synthetic, seeded); resident in HBM before timing
    H_host = S.channels(spec, trials=trials)
    tdt = torch.complex64 if spec.dtype == "c64" else torch.complex128
    H_pin = torch.from_numpy(H_host).pin_memory()
    del H_host
    H_dev = H_pin.to(dev)
    noise = torch.from_numpy(np.ascontiguousarray(
        np.broadcast_to(S.noise_vector(spec), (B, K)))).to(dev)
    cfg_wb = TrajectoryConfig(alpha=spec.alpha, eta=eta, k_init=spec.k_init, p=spec.p,
                              i_max=spec.i_max)
    cfg_full = TrajectoryConfig(alpha=spec.alpha, eta=None)
    L = T * TrajectoryRunner(B, K, Nn, tdt, cfg_wb, dev).normals_per_step_max()
    # sketch streams: the harness's per-(method, trial) PCG64 Generators
    # (harness.py:88-92), reproduced on the device; each step regenerates its
    # window from the stream start so every timed step does identical work
    streams = DeviceOmegaStreams.for_method(spec.seed, eta, trials, dev)
    stream = torch.cuda.current_stream(dev)

    # LRZ_RNG_PRIO=-1 puts the sketch RNG on a high-priority stream (its CTAs are
    # dispatched first as SM slots free up beside the Gram)
    rng_stream = torch.cuda.Stream(dev, priority=int(os.environ.get("LRZ_RNG_PRIO", "0")))

    def one(cfg, prof=None, Hd=H_dev, st=streams, sl=slice(None), sync=True):
        nb = Hd.shape[0]
        rn = TrajectoryRunner(nb, K, Nn, tdt, cfg, dev)
        rn.prof = prof
        om = None
        if cfg.eta is not None:
            st.raw.zero_()
            if prof is not None:   # stage profile: serialised so the RNG's own time is seen
                e0 = rn._ev()
                om = st.window(L)
                rn._stage("omega_rng", e0)
            else:                  # the step: Omega generated on a side stream under the Gram
                om = st.window(L, stream=rng_stream)
        return rn.run_chunk(Hd, noise[sl], om, omega_ready=st.ready, sync=sync)

    use_graph = not args.no_graph

    def capture(cfg):
        """The whole step (fresh runner, Omega window, Gram ... rate) as one CUDA
        graph; the verifier flags of every replay accumulate on the device."""
        acc = torch.zeros(2, dtype=torch.int32, device=dev)
        g = torch.cuda.CUDAGraph()
        torch.cuda.synchronize(dev)
        with torch.cuda.graph(g):
            r = one(cfg, sync=False)
            if r.flags is not None:
                acc.add_(r.flags)
        torch.cuda.synchronize(dev)
        return g, r, acc

    def timed(cfg, steps, graph=None):
        barrier()
        torch.cuda.synchronize(dev)
        l0 = ops.LAUNCHES[0]
        last = one(cfg)                      # eager step: kernel count, verified results
        torch.cuda.synchronize(dev)
        n_launch = ops.LAUNCHES[0] - l0
        if graph is not None:
            g, gres, acc = graph
            acc.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        e0.record(stream)
        for _ in range(steps):
            if graph is not None:
                g.replay()
            else:
                last = one(cfg)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        if graph is not None:
            if int(acc.abs().sum().item()):
                raise RuntimeError("graph replay left unverified arSVD steps; rerun with --no-graph")
            # the replayed results equal the eager step's (same inputs, same streams)
            if not torch.equal(gres.method, last.method) or \
                    not torch.allclose(gres.rates, last.rates, rtol=0, atol=0):
                raise RuntimeError("graph replay differs from the eager step")
            last = gres
        ms = max_over_ranks(e0.elapsed_time(e1)) / steps
        return ms, n_launch, last

    for _ in range(args.warmup):
        one(cfg_wb)
        one(cfg_full)
    graphs = {}
    if use_graph:
        graphs = {"wb": capture(cfg_wb), "full": capture(cfg_full)}
        for g, _, _ in graphs.values():     # warm replays
            g.replay()
        torch.cuda.synchronize(dev)
    with Clocks(local) as clk:
        ms_wb, launches, last = timed(cfg_wb, args.steps, graphs.get("wb"))
        ms_full, launches_full, _ = timed(cfg_full, args.steps, graphs.get("full"))
    # stage split: separate eager steps with CUDA events between stages (serialised RNG)
    prof = []
    n_prof = min(args.steps, 3)
    for _ in range(n_prof):
        one(cfg_wb, prof)
    torch.cuda.synchronize(dev)
    updates = B * T
    value = world * updates / (ms_wb / 1e3)
    value_full = world * updates / (ms_full / 1e3)

    # per-stage device time over the timed WB steps (CUDA events on the stream)
    stage_ms = {}
    for name, a, b in prof:
        stage_ms[name] = stage_ms.get(name, 0.0) + a.elapsed_time(b)
    stage_ms = {k: v / n_prof for k, v in stage_ms.items()}
    if world > 1:
        # one gather of the per-trial results, merged by trial index
        from paper_2512_16543_b200.dist import gather_results
        merged = gather_results({"rates": last.rates.cpu().numpy(),
                                 "k_est": last.k_est.cpu().numpy(),
                                 "method": last.method.cpu().numpy()},
                                trials, world * B, device=dev)
        assert merged["rates"].shape == (world * B, T)
    method = last.method.cpu().numpy()
    k_est = last.k_est.cpu().numpy()
    iters = last.iters.cpu().numpy()
    wb_steps = int((method == 1).sum())
    k_mean = float(k_est[method == 1].mean()) if wb_steps else 0.0
    hist = {int(i): int(c) for i, c in zip(*np.unique(iters[iters > 0], return_counts=True))}
    model = stage_model(spec, T, B, k_mean, hist, wb_steps)
    peaks = measured_peaks(torch, dev)
    mp_path = ROOT / "MEASURED_PEAKS.json"
    hbm = json.loads(mp_path.read_text())["hbm_gbs"] if mp_path.exists() else 6650.0
    fpk = peaks["fp64"] if spec.dtype == "c128" else peaks["fp32"]
    # dominant kernel: a stage of n main kernels is credited stage_ms / n per kernel
    # (arSVD = sketch GEMM + screen; the launch list in profiles/ has the split),
    # so a single-kernel stage longer than that wins
    per_kernel = {k: stage_ms[k] / STAGE_MAIN_KERNELS.get(k, 1) for k in stage_ms if k in model}
    dom = max(per_kernel, key=lambda k: per_kernel[k])
    flops, byts = model[dom]
    launches_dom = {"arsvd": max(last.spec_passes, 1), "gram_delta": 2}.get(dom, 1)
    t = stage_ms[dom] / 1e3
    t_f, t_b = flops / (fpk * 1e12), byts / (hbm * 1e9)
    if t_f >= t_b:
        roof = {"bound": "tensor", "achieved": flops / t / 1e12, "peak": fpk, "unit": "TFLOP/s",
                "peak_source": f"measured now: cuBLAS {'DGEMM' if spec.dtype == 'c128' else 'SGEMM (TF32 off)'} 8192^3 via torch.matmul (MEASURED_PEAKS.json has no fp64/fp32 entry)"}
    else:
        roof = {"bound": "hbm", "achieved": byts / t / 1e9, "peak": hbm, "unit": "GB/s",
                "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["kernel"] = dom
    roof["kernels"] = [frag for frag, _ in STAGE_KERNELS.get(dom, [])]
    roof["launches_per_step"] = launches_dom
    tr = stage_traffic(dom, spec)
    roof["traffic"] = tr["bytes_per_step"] if tr else None
    roof["traffic_note"] = (tr["source"] + "; per step, like 'algorithmic' (compulsory "
                            "bytes: H in, W out, A^-1 and G in for the precoder; dA + Omega "
                            "for the arSVD front end)") if tr else None
    roof["algorithmic"] = {"flops_per_step": flops, "bytes_per_step": byts}
    all_stages = {}
    for k, v in stage_ms.items():
        if k in model and v > 0:
            f, b_ = model[k]
            # roofline fraction of the stage: the slower of its flops at the FP64 (c64:
            # FP32) peak and its compulsory bytes at HBM bandwidth, over its time
            tb = max(f / (fpk * 1e12), b_ / (hbm * 1e9))
            all_stages[k] = {"ms": v, "tflops": f / (v / 1e3) / 1e12, "gbs": b_ / (v / 1e3) / 1e9,
                             "bound": "tensor" if f / (fpk * 1e12) >= b_ / (hbm * 1e9) else "hbm",
                             "frac": tb / (v / 1e3)}
        else:
            all_stages[k] = {"ms": v}

    # ---- e2e: host (pinned) channels -> device -> results back, every step.
    # Trials are split into groups, each with its own device buffer; all H2D
    # copies are queued back to back on a copy stream (PCIe is the bound) and
    # group g's compute starts as soon as its copy lands.  Groups run without
    # a host round trip (sync=False); their verifier flags accumulate on the
    # device and are checked after the timed region.  Omega is generated on
    # the device.
    e2e = None
    if not args.no_e2e:
        ng = 8 if B % 8 == 0 else 1
        bs = B // ng
        gstreams = [DeviceOmegaStreams.for_method(spec.seed, eta, trials[g * bs:(g + 1) * bs], dev)
                    for g in range(ng)]
        bufs = [torch.empty((bs,) + tuple(H_dev.shape[1:]), dtype=H_dev.dtype, device=dev)
                for _ in range(ng)]
        copy_s = torch.cuda.Stream(dev)
        outs_pin = {}
        acc = torch.zeros(2, dtype=torch.int32, device=dev)
        n_e2e = max(2, min(args.steps, 3))

        def e2e_step():
            copied = []
            for g in range(ng):
                with torch.cuda.stream(copy_s):
                    copy_s.wait_stream(stream)        # previous step's readers of bufs[g]
                    bufs[g].copy_(H_pin[g * bs:(g + 1) * bs], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(copy_s)
                    copied.append(ev)
            for g in range(ng):
                stream.wait_event(copied[g])
                r = one(cfg_wb, None, bufs[g], gstreams[g], slice(g * bs, (g + 1) * bs),
                        sync=False)
                if r.flags is not None:
                    acc.add_(r.flags)
                for name in ("rates", "per_ut", "method", "k_est"):
                    t = getattr(r, name)
                    key = (name, g)
                    if key not in outs_pin:
                        outs_pin[key] = torch.empty(t.shape, dtype=t.dtype).pin_memory()
                    outs_pin[key].copy_(t, non_blocking=True)

        e2e_step()
        barrier()
        torch.cuda.synchronize(dev)
        acc.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(n_e2e):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        if int(acc.abs().sum().item()):
            raise RuntimeError("e2e groups left unverified arSVD steps")
        ms_e2e = max_over_ranks(e0.elapsed_time(e1)) / n_e2e
        d2h = sum(t.numel() * t.element_size() for t in outs_pin.values())
        e2e = {"value": world * updates / (ms_e2e / 1e3), "unit": "updates/s",
               "h2d_bytes_per_step": H_pin.numel() * H_pin.element_size(),
               "d2h_bytes_per_step": d2h, "ms_per_step": ms_e2e,
               "path": "TrajectoryRunner.run_chunk (public batched API over the C ABI): pinned "
                       f"host H copied in per step in {ng} trial groups queued back to back "
                       "on a copy stream, each group's compute starting when its copy lands; "
                       "Omega generated on the device from the harness's PCG64 streams; "
                       "rates/per-UT rates/method/k_est copied out"}
        del bufs

    # ---- c64 side measurement (same workload, complex64 inputs)
    extra = None
    if not args.no_extra and spec.dtype == "c128":
        H64 = H_dev.to(torch.complex64)
        torch.cuda.synchronize(dev)

        def one64(cfg):
            rn = TrajectoryRunner(B, K, Nn, torch.complex64, cfg, dev)
            om = None
            if cfg.eta is not None:
                streams.raw.zero_()
                om = streams.window(L)
            return rn.run_chunk(H64, noise, om)

        for cfg in (cfg_wb, cfg_full):
            one64(cfg)
        res64 = {}
        for name, cfg in (("wb", cfg_wb), ("full", cfg_full)):
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                one64(cfg)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            res64[name] = world * updates / (max_over_ranks(e0.elapsed_time(e1)) / args.steps / 1e3)
        extra = {"c64_wb_updates_per_s": res64["wb"], "c64_full_updates_per_s": res64["full"]}
        del H64

    # ---- the reference's own LEO campaign (hybrid beams), SURVEY 8(f) #3/#4
    leo = None
    if not args.no_extra:
        # the campaign allocates its own multi-GB chunk buffers: hand back the
        # graph pools and cached blocks of the C2 measurements first
        graphs.clear()
        torch.cuda.synchronize(dev)
        torch.cuda.empty_cache()
        leo = leo_side(args, dev, world, max_over_ranks)

    # ---- CPU baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cores = _cores()
        n_trials = min(B, cores)
        with _cpu_pool(cores, spec) as pool:
            v_cpu = cpu_rate(spec, eta, n_trials, pool)
        cpu = {"value": v_cpu, "unit": "updates/s", "cores": cores, "kind": "port",
               "sample": f"{n_trials} trials x {spec.T} steps of the WB-arSVD method, one trial "
                         f"per worker process, oracle port with F_RF = I_N verbatim, "
                         f"BLAS 1 thread/worker"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "updates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_wb,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": spec.dtype + (" (fp64 arithmetic)" if spec.dtype == "c128" else
                                   " (fp32 N-sized products, fp64 K x K chain)"),
            "data": "synthetic (SURVEY.md 8(d) seeded Rician drift channels; the reference has "
                    "no public dataset)",
            "config": {"workload": workload_desc(spec, eta),
                       "parallelism": f"trials sharded over {world} GPU(s)",
                       "l2": "inputs larger than L2 (H = %.2f GB per GPU), no flush needed"
                             % (H_pin.numel() * H_pin.element_size() / 1e9),
                       "updates_per_step": updates * world},
            "full_inverse": {"value": value_full, "unit": "updates/s", "ms_per_step": ms_full,
                             "gpu_launches": launches_full},
            "roofline": roof,
            "stages": all_stages,
            "peaks_measured": peaks,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "spec_passes": last.spec_passes,
            "omega": "generated on the device each step (PCG64 + numpy ziggurat, the "
                     "harness's per-(method, trial) streams; bit-exact except ulp-level "
                     "log1p tail values)",
            "method_counts": {"full": int((method == 0).sum()), "woodbury": wb_steps,
                              "none": int((method == 2).sum())},
            "clocks": clk.summary(),
        }
        if extra:
            line["c64"] = extra
        if leo:
            line["leo_campaign"] = leo
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
