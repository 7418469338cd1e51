"""The reference's default LEO campaign (ScenarioConfig defaults: K = N_RF = 16,
16x16 array, 2400 snapshots, 50 passes, conventional + eta 0.9/0.8/0.65) on
one GPU, timed with CUDA events, next to the CPU oracle port on the host cores.

    python scripts/leo_campaign.py [--mc 50] [--chunk 600] [--cpu-trials 16 --cpu-steps 120]

Prints one JSON line: precoder updates/s (all methods) and passes/s, the
comparison table, and the CPU sample rate.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2512_16543_b200 import leo as L  # noqa: E402


def _cpu_job(args):
    cfg_kw, trial, steps = args
    from oracle import leo as OL
    cfg = L.ScenarioConfig(**cfg_kw)
    etas = sorted(set(cfg.eta_list), reverse=True)
    specs = [(OL.label_of(None), None)] + [(OL.label_of(e), e) for e in etas]
    t0 = time.perf_counter()
    OL.sweep_trial(cfg, specs, trial, cfg.seed, steps=steps)
    return time.perf_counter() - t0


def cpu_rate(cfg_kw, trials, steps, cores, n_methods):
    import multiprocessing as mp
    for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[v] = "1"
    ctx = mp.get_context("spawn")
    with ctx.Pool(cores) as pool:
        pool.map(_cpu_job, [(cfg_kw, 0, 2)] * cores)          # warm-up
        t0 = time.perf_counter()
        pool.map(_cpu_job, [(cfg_kw, t, steps) for t in range(trials)])
        wall = time.perf_counter() - t0
    return trials * steps * n_methods / wall, wall


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mc", type=int, default=50)
    ap.add_argument("--chunk", type=int, default=600)
    ap.add_argument("--cpu-trials", type=int, default=16)
    ap.add_argument("--cpu-steps", type=int, default=120)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    cfg = L.ScenarioConfig(mc_runs=args.mc).validate()
    n_methods = 1 + len(set(cfg.eta_list))
    dev = torch.device("cuda", 0)
    L.run_campaign(cfg.with_(mc_runs=2, pass_s=10.0), chunk=args.chunk, device=dev)   # warm-up
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    e0.record()
    res = L.run_campaign(cfg, chunk=args.chunk, device=dev, collect_decisions=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    wall = time.perf_counter() - w0
    updates = cfg.mc_runs * cfg.n_snapshots * n_methods
    line = {"workload": "leo_default_campaign", "mc_runs": cfg.mc_runs,
            "n_snapshots": cfg.n_snapshots, "methods": res.labels,
            "gpu_ms": ms, "gpu_wall_s": wall, "updates_per_s": updates / (ms / 1e3),
            "passes_per_s": cfg.mc_runs / (ms / 1e3),
            "table": [[r.method_label, r.savings_pct, r.degradation_pct] for r in res.table.rows],
            "mean_k_est": res.mean_k_est, "method_counts": res.method_counts,
            "gpu": torch.cuda.get_device_name(0)}
    if not args.no_cpu:
        cores = len(os.sched_getaffinity(0))
        kw = {k: getattr(cfg, k) for k in L.ScenarioConfig.__dataclass_fields__}
        v, w = cpu_rate(kw, args.cpu_trials, args.cpu_steps, cores, n_methods)
        line["cpu_baseline"] = {"value": v, "unit": "updates/s", "cores": cores, "kind": "port",
                                "sample": f"{args.cpu_trials} passes x first {args.cpu_steps} "
                                          f"snapshots x {n_methods} methods", "wall_s": w}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
