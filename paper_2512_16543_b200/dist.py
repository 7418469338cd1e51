"""Multi-GPU trial sharding.

Trials are independent Monte-Carlo passes, so N GPUs split the trial range
(one process per GPU, torch.distributed) with no exchange on the data path;
the per-trial results (rates, k_est, method, cost, normals consumed) are
gathered once at the end and merged by trial index, which makes a sharded run
bit-identical to a serial one (the property the reference harness states for
its process pool, harness.py:9-10,336-356).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

FIELDS = ("rates", "per_ut", "method", "k_est", "iters", "cost", "consumed")


def shard_trials(n_trials: int, rank: int, world: int) -> list[int]:
    """Contiguous trial block of `rank`; the first n % world ranks get one extra."""
    base, extra = divmod(n_trials, world)
    start = rank * base + min(rank, extra)
    return list(range(start, start + base + (1 if rank < extra else 0)))


def gather_results(local: dict, trials: list[int], n_trials: int, group=None,
                   device=None) -> dict | None:
    """All-gather per-trial arrays (leading dim = local trial count) from every
    rank and merge them by trial index.  Returns the merged dict on every rank.
    `local[name]` are numpy arrays; one collective per field plus one for the
    trial ids (padding to the largest shard)."""
    world = dist.get_world_size(group)
    dev = torch.device("cpu") if device is None else device
    cnt = torch.tensor([len(trials)], dtype=torch.int64, device=dev)
    counts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(counts, cnt, group=group)
    mx = int(max(int(c.item()) for c in counts))

    def pad(a: np.ndarray) -> torch.Tensor:
        t = torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        if t.shape[0] < mx:
            t = torch.cat([t, torch.zeros((mx - t.shape[0],) + tuple(t.shape[1:]),
                                          dtype=t.dtype, device=dev)])
        return t

    ids = pad(np.asarray(trials, dtype=np.int64))
    all_ids = [torch.empty_like(ids) for _ in range(world)]
    dist.all_gather(all_ids, ids, group=group)
    order = []
    for r in range(world):
        n = int(counts[r].item())
        order.extend(int(x) for x in all_ids[r][:n].cpu().numpy())
    if sorted(order) != list(range(n_trials)):
        raise ValueError("trial shards do not cover 0..n_trials-1 exactly once")
    out = {}
    for name, a in local.items():
        t = pad(np.asarray(a))
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t, group=group)
        merged = np.empty((n_trials,) + tuple(t.shape[1:]), dtype=np.asarray(a).dtype)
        for r in range(world):
            n = int(counts[r].item())
            ids_r = all_ids[r][:n].cpu().numpy()
            merged[ids_r] = parts[r][:n].cpu().numpy()
        out[name] = merged
    return out
