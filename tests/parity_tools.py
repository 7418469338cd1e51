"""Per-step parity replay of GPU trajectories against the oracle sweep
(test infrastructure; imported only by tests/).

SURVEY.md A.4: WB parity is a chained comparison -- one rank flip diverges
the rest of the trial -- so each trial is compared step by step up to its
first *genuine* near-threshold tie (oracle decision margin below a
dtype-scaled bound), never skipped as a whole.  Every step
before the stop is checked in full: k_est, method and normals consumed
exactly; A^-1 and the power-normalised precoder F_BB (W) within the
north-star tolerance (relative Frobenius); per-step sum-rates within the
rate tolerance.  A mismatch at a step whose margin is not a tie fails.

The oracle replays run in spawned worker processes (one BLAS thread each,
like harness.py:284-293); their A^-1 / F_BB sequences come back through .npy
files so the large configs (C5: 100 x 4096 x 256 complex per trial) do not
travel through a pipe.
"""

from __future__ import annotations

import dataclasses
import json
import multiprocessing as mp
import os
import tempfile
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]

# near-tie bounds on the oracle's decision margin |cum - target| / target:
# complex64 energies carry ~1e-6 relative error (fp32 Gram correction), complex128 ~1e-13
TIE_BOUND = {"c64": 1e-4, "c128": 1e-9}
TOL = {"c64": 1e-4, "c128": 1e-10}      # north_star: A^-1 / W relative Frobenius
RATE_TOL = {"c64": 1e-4, "c128": 1e-9}  # per-step sum-rate, relative


def _oracle_job(job):
    """Worker: one trial of one method through the oracle sweep."""
    spec_kw, trial, eta, T, out_dir = job
    try:
        import threadpoolctl
        threadpoolctl.threadpool_limits(1)
    except Exception:
        pass
    from oracle import port, sweep
    from paper_2512_16543_b200 import scenario as S
    spec = S.ScenarioSpec(**spec_kw)
    H = S.trial_channels(spec, trial, 0, T)
    if spec.dtype == "c64":
        H = H.astype(np.complex64)
    cfg = None if eta is None else port.Cfg(eta, spec.k_init, spec.p, spec.i_max)
    sk = None if eta is None else np.random.default_rng(
        S.stream_seed(spec.seed, S.method_label(eta), trial))
    rec = sweep.sweep_trial(H, spec.alpha, S.noise_vector(spec), 1.0, cfg, sk, keep_state=True)
    tag = f"{spec.name}_{spec.dtype}_{spec.cap}_{spec.tol:g}_{eta}_{trial}"
    a_path = os.path.join(out_dir, tag + "_Ainv.npy")
    f_path = os.path.join(out_dir, tag + "_FBB.npy")
    np.save(a_path, np.stack(rec.A_inv))
    np.save(f_path, np.stack(rec.F_BB))
    small = {k: getattr(rec, k) for k in ("rates", "method", "k_est", "consumed", "iters",
                                          "margin", "margin_min", "fallback")}
    return small, a_path, f_path


def oracle_replays(jobs, workers: int | None = None):
    """jobs: list of (spec, trial, eta, T).  Returns a list of (small dict,
    A_inv path, F_BB path), in job order."""
    out_dir = tempfile.mkdtemp(prefix="lrz_parity_")
    packed = [(dataclasses.asdict(s), t, e, T, out_dir) for s, t, e, T in jobs]
    n = workers or min(len(packed), max(1, (os.cpu_count() or 2) - 1))
    env = {k: os.environ.get(k) for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS",
                                          "MKL_NUM_THREADS")}
    for k in env:
        os.environ[k] = "1"
    try:
        with mp.get_context("spawn").Pool(n) as pool:
            return pool.map(_oracle_job, packed, chunksize=1)
    finally:
        for k, v in env.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _rel(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def compare_trial(gpu, b, ref, a_path, f_path, dtype, label):
    """Per-step comparison of GPU trial row b with one oracle replay.
    Returns a summary dict; raises AssertionError on a non-tie mismatch or a
    tolerance violation before the stop step."""
    T = len(ref["k_est"])
    tol, rtol, tie_b = TOL[dtype], RATE_TOL[dtype], TIE_BOUND[dtype]
    stop, tie = T, False
    for t in range(T):
        same = (gpu.k_est[b, t] == ref["k_est"][t] and gpu.method[b, t] == ref["method"][t]
                and gpu.consumed[b, t] == ref["consumed"][t])
        if not same:
            m = float(min(ref["margin_min"][t], ref["margin"][t]))
            assert m < tie_b, (
                f"{label}: step {t} differs and is not a tie (oracle margin {m:.3e}): "
                f"k {gpu.k_est[b, t]} vs {ref['k_est'][t]}, method {gpu.method[b, t]} vs "
                f"{ref['method'][t]}, consumed {gpu.consumed[b, t]} vs {ref['consumed'][t]}")
            stop, tie = t, True
            break
    A_ref = np.load(a_path, mmap_mode="r")
    F_ref = np.load(f_path, mmap_mode="r")
    a_err = w_err = r_err = 0.0
    for t in range(stop):
        a_err = max(a_err, _rel(gpu.A_inv[b, t], A_ref[t]))
        w_err = max(w_err, _rel(gpu.W[b, t], F_ref[t]))
        r_err = max(r_err, abs(gpu.rates[b, t] / ref["rates"][t] - 1.0))
    del A_ref, F_ref
    for pth in (a_path, f_path):
        try:
            os.remove(pth)
        except OSError:
            pass
    assert a_err < tol, f"{label}: A_inv rel err {a_err:.3e} over {stop} steps"
    assert w_err < tol, f"{label}: W (F_BB) rel err {w_err:.3e} over {stop} steps"
    assert r_err < rtol, f"{label}: sum-rate rel err {r_err:.3e} over {stop} steps"
    return {"label": label, "steps": T, "compared": stop, "tie_stop": tie,
            "A_inv_err": a_err, "W_err": w_err, "rate_err": r_err,
            "woodbury_steps": int(np.sum(ref["method"][:stop] == 1)),
            "k_max": int(np.max(ref["k_est"][:stop])) if stop else 0,
            "fallback_steps": int(np.sum(ref["fallback"][:stop]))}


def record(rows, name: str):
    """Append per-trial summaries to gpurun_out/<name>.json (tie-rate table)."""
    out = ROOT / "gpurun_out"
    out.mkdir(exist_ok=True)
    path = out / f"{name}.json"
    old = json.loads(path.read_text()) if path.exists() else []
    path.write_text(json.dumps(old + rows, indent=1))
