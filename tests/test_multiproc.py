"""The N > 1 path on CPU: world_size-2 process group over gloo (127.0.0.1).

Frames shard across ranks with no collective on the data path
(paper_2001_07979_b200/shard.py).  Each rank decodes its
contiguous shard -- here with the oracle standing in for the GPU decoder,
since this container has no GPU -- and the results gathered to rank 0 must
equal the reference's golden outputs for the whole stream; the timing
reduction bench.py uses must give sum-of-work / max-of-time.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2001_07979_b200.shard import shard_range


def test_shard_range_covers_stream_once():
    for total in (0, 1, 31, 64, 65536, 1000):
        for world in (1, 2, 3, 8):
            spans = [shard_range(total, world, r) for r in range(world)]
            got = [i for lo, hi in spans for i in range(lo, hi)]
            assert got == list(range(total))
            assert all(hi - lo <= -(-total // world) for lo, hi in spans)
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


class _OracleDecoder:
    """BatchDecoder.decode stand-in (test infrastructure): the oracle."""

    def __init__(self, ensemble):
        import oracle
        from paper_2001_07979_b200.matrix import stacked_layout

        self.og = oracle.OracleGraph(stacked_layout(ensemble))

    def decode(self, noisy, syn, e):
        import oracle
        from paper_2001_07979_b200.decoder import BatchResult

        corrected, conv, iters, mism = oracle.decode_batch(self.og, noisy, syn, e, threads=2)
        return BatchResult(corrected, conv, iters, mism.astype(np.int32), 0)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from conftest import _ens, load_golden
    from paper_2001_07979_b200.shard import decode_shard, gather_results, reduce_work_time

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ens = _ens("cfg1")
        g = load_golden("golden_cfg1.npz")
        noisy, syn = g["e070_noisy"], g["e070_syn"]
        lo, hi, res = decode_shard(_OracleDecoder(ens), noisy, syn, 0.07, world, rank)
        full = gather_results(lo, hi, res, ens.n)
        work, times = reduce_work_time([float(hi - lo)], [1.0 + rank], device=torch.device("cpu"))
        if rank == 0:
            ok = (np.array_equal(full["iterations"], g["e070_iterations"])
                  and np.array_equal(full["converged"], g["e070_converged"])
                  and np.array_equal(full["corrected"][g["e070_converged"]],
                                     g["e070_corrected"][g["e070_converged"]]))
            q.put((ok, work, times, full["iterations"].shape[0]))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_shard_decode_and_gather():
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent))
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    ok, work, times, frames = q.get()
    assert ok
    assert frames == 32
    assert work == [32.0]          # frames summed over ranks
    assert times == [2.0]          # max over ranks
