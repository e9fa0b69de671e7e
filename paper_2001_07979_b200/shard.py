"""Frame sharding across ranks.

Frames are independent (decoder.py:19-23), so a stream of F
frames is split into contiguous shards of ceil(F / world) frames, one per rank
(one process per GPU), each decoded with its own ensemble replica.  There is
no collective on the data path: results come back to the host of each rank
and are gathered to rank 0 (pickled rows over the process group -- gloo on
CPU, NCCL under torchrun; it is the reference's "gather results" step, not
part of decoding).  Timing is reduced as sum of work / max of time over ranks.
"""

from __future__ import annotations

import numpy as np


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous frame range [lo, hi) of `rank` out of `world` (ceil split;
    trailing ranks may get fewer or no frames)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world size {world}")
    per = -(-total // world)
    lo = min(total, rank * per)
    return lo, min(total, lo + per)


def decode_shard(decoder, noisy_rows, syn_rows, e, world: int, rank: int):
    """Decode this rank's shard of the frame stream.  `decoder` is anything
    with the BatchDecoder.decode(noisy, syn, e) signature.  Returns
    (lo, hi, result)."""
    lo, hi = shard_range(noisy_rows.shape[0], world, rank)
    ev = np.asarray(e, dtype=np.float64)
    e_shard = ev if ev.ndim == 0 or ev.size == 1 else ev[lo:hi]
    res = decoder.decode(noisy_rows[lo:hi], syn_rows[lo:hi], e_shard) if hi > lo else None
    return lo, hi, res


def gather_results(lo: int, hi: int, res, n: int, group=None):
    """Gather every rank's (lo, hi, per-frame outputs) to rank 0 and assemble
    the stream's arrays in frame order.  Returns a dict on rank 0, None
    elsewhere."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    payload = None
    if res is not None:
        payload = (lo, hi, np.asarray(res.corrected), np.asarray(res.converged, dtype=bool),
                   np.asarray(res.iterations), np.asarray(res.mismatches))
    items = [None] * world
    dist.all_gather_object(items, payload, group=group)
    if dist.get_rank(group) != 0:
        return None
    parts = sorted((p for p in items if p is not None), key=lambda p: p[0])
    return {
        "corrected": np.concatenate([p[2] for p in parts]),
        "converged": np.concatenate([p[3] for p in parts]),
        "iterations": np.concatenate([p[4] for p in parts]),
        "mismatches": np.concatenate([p[5] for p in parts]),
        "n": n,
    }


def reduce_work_time(work: list[float], times: list[float], device=None, group=None):
    """Whole-job aggregation used by bench.py: sum of per-rank work counters,
    max of per-rank times (device-timed)."""
    import torch
    import torch.distributed as dist

    w = torch.tensor(work, dtype=torch.float64, device=device)
    t = torch.tensor(times, dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(w, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return w.tolist(), t.tolist()
