"""updates/s for every BASELINE config (C1-C5) on one GPU, next to the CPU
reference algorithm on the host cores.

GPU: the everything-on-device campaign (channels synthesised per time chunk,
device sketch streams, batched runner), full trial count and T of each
config, timed with CUDA events after one untimed warm-up pass of the same
config (the time includes the host-side parameter draws of every trial).  CPU: the oracle port
on all cores (one trial per worker, BLAS 1 thread) on a bounded sample of
trials x steps of the same config.

    python scripts/all_configs.py [--out profiles/r01_configs.json] [--quick]
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2512_16543_b200 import scenario as S  # noqa: E402
from paper_2512_16543_b200.trajectory import run_campaign_device  # noqa: E402

RUNS = [
    # (label, spec overrides, chunk T)
    ("C1", dict(), 50),
    ("C2", dict(dtype="c128"), 200),
    ("C2", dict(dtype="c64"), 200),
    ("C2", dict(dtype="c128", snr_db=0.0), 200),
    ("C2", dict(dtype="c128", snr_db=20.0), 200),
    ("C3", dict(), 50),
    ("C4", dict(cap=8, tol=1e-3), 8),
    ("C4", dict(cap=32, tol=1e-3), 8),
    ("C4", dict(cap=16, tol=1e-2), 8),
    ("C5", dict(dtype="c64"), 10),
    ("C5", dict(dtype="c128"), 5),
]


def gpu_rate(spec, eta, chunk, dev):
    # warm-up: one full pass (allocations, library first calls), then the timed pass
    run_campaign_device(spec, eta, range(spec.B), dev, chunk=chunk, keep=True)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = run_campaign_device(spec, eta, range(spec.B), dev, chunk=chunk, keep=True)
    e1.record()
    torch.cuda.synchronize(dev)
    wall = time.perf_counter() - t0
    ms = e0.elapsed_time(e1)
    meth = res.method[:, 1:]
    return {"updates_per_s": spec.B * spec.T / (ms / 1e3), "wall_s": wall,
            "method_frac": {"full": float((meth == 0).mean()), "woodbury": float((meth == 1).mean()),
                            "none": float((meth == 2).mean())},
            "mean_k_est": float(res.k_est[:, 1:].mean()), "spec_passes": res.spec_passes[:4],
            "mean_sum_rate": float(res.rates.mean())}


def cpu_rate(spec, eta, pool, cores, steps):
    sample = spec.with_(T=steps)
    n = min(spec.B, cores)
    v = bench.cpu_rate(sample, eta, n, pool)
    return {"updates_per_s": v, "sample": f"{n} trials x {steps} steps", "cores": cores}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "profiles" / "r01_configs.json"))
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    cores = bench._cores()
    rows = []
    pool = None
    for label, kw, chunk in RUNS:
        spec = S.CONFIGS[label].with_(**kw)
        if args.quick:
            spec = spec.with_(B=min(spec.B, 16), T=min(spec.T, 2 * chunk))
        row = {"config": label, "spec": {k: v for k, v in dataclasses.asdict(spec).items()
                                         if k not in ("name",)},
               "eta": spec.eta, "i_max": spec.i_max}
        for name, eta in (("wb_arsvd", spec.eta), ("full", None)):
            row[f"gpu_{name}"] = gpu_rate(spec, eta, chunk, dev)
            torch.cuda.empty_cache()
        if not args.no_cpu:
            if pool is None:
                pool = bench._cpu_pool(cores, spec)
            steps = {"C1": 50, "C2": 40, "C3": 6, "C4": 3, "C5": 2}[label]
            row["cpu_wb_arsvd"] = cpu_rate(spec, spec.eta, pool, cores, steps)
        rows.append(row)
        print(json.dumps({"config": label, **{k: row[k] for k in row if k.startswith(("gpu", "cpu"))}}),
              flush=True)
    if pool is not None:
        pool.close()
    Path(args.out).parent.mkdir(exist_ok=True)
    Path(args.out).write_text(json.dumps({"gpu": torch.cuda.get_device_name(0), "rows": rows},
                                         indent=1))


if __name__ == "__main__":
    main()
