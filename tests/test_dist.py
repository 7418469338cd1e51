"""Trial sharding across ranks (world_size 2, gloo, CPU): the merged sharded
run is bit-identical to the serial run (harness.py:9-10)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2512_16543_b200.dist import shard_trials


def test_shard_trials_cover_exactly_once():
    for n, w in [(64, 1), (64, 2), (65, 2), (7, 3), (3, 8)]:
        got = [t for r in range(w) for t in shard_trials(n, r, w)]
        assert got == list(range(n))
        sizes = [len(shard_trials(n, r, w)) for r in range(w)]
        assert max(sizes) - min(sizes) <= 1


def _sweep(spec, eta, trials):
    from oracle import port, sweep
    from paper_2512_16543_b200 import scenario as S
    out = {k: [] for k in ("rates", "method", "k_est", "consumed")}
    for b in trials:
        H = S.trial_channels(spec, b)
        sk = np.random.default_rng(S.stream_seed(spec.seed, S.method_label(eta), b))
        rec = sweep.sweep_trial(H, spec.alpha, S.noise_vector(spec), 1.0,
                                port.Cfg(eta, spec.k_init, spec.p, spec.i_max), sk)
        for k in out:
            out[k].append(getattr(rec, k))
    return {k: np.stack(v) for k, v in out.items()}


def _worker(rank, world, port_no, q):
    import torch.distributed as dist
    from paper_2512_16543_b200 import scenario as S
    from paper_2512_16543_b200.dist import gather_results
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    spec = S.C1.with_(B=5, T=8)
    mine = shard_trials(spec.B, rank, world)
    merged = gather_results(_sweep(spec, 0.9, mine), mine, spec.B)
    if rank == 0:
        q.put({k: v for k, v in merged.items()})
    dist.barrier()
    dist.destroy_process_group()


def test_gather_matches_serial_world2():
    from paper_2512_16543_b200 import scenario as S
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port_no = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port_no, q)) for r in range(2)]
    for p in procs:
        p.start()
    merged = q.get(timeout=240)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    spec = S.C1.with_(B=5, T=8)
    serial = _sweep(spec, 0.9, range(spec.B))
    for k in serial:
        assert np.array_equal(merged[k], serial[k]), k
