"""Streams: device frame generation, the pipelined host path for batches
larger than the workspace, and the sharded multi-rank path on the GPU.

* mbp_frames_generate_device == the reference's numpy frame streams
  (bench._frame_inputs, bench.py:123-130), bit for bit;
* mbp_decode_batch with batch > capacity (two-slot staging ring: H2D of
  chunk c+1 || decode c || D2H c-1) == the device path, per frame;
* two ranks (gloo, one GPU) each decode their contiguous shard with
  BatchDecoder; the gathered stream equals the reference's golden outputs.
"""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2001_07979_b200 import BatchDecoder
from paper_2001_07979_b200.channel import make_frames, make_frames_device

pytestmark = pytest.mark.gpu
HERE = Path(__file__).resolve().parent


@pytest.mark.parametrize("n,e,seed,path,start,frames", [
    (65536, 0.03, 0, (), 0, 40),
    (65536, 0.05, 0, (), 60000, 7),
    (4096, 0.07, 0, (7,), 0, 33),
    (1000, 0.09, 3, (2, 99), 5, 5),
    (37, 0.25, 2**33 + 1, (1,), 2**32 + 3, 3),
])
def test_device_generator_equals_numpy_streams(n, e, seed, path, start, frames):
    import torch

    ref = make_frames(n, e, frames, seed=seed, path=path, start=start)
    keys, noisy = make_frames_device(n, e, frames, seed=seed, path=path, start=start)
    torch.cuda.synchronize()
    assert np.array_equal(keys.cpu().numpy(), ref.keys)
    assert np.array_equal(noisy.cpu().numpy(), ref.noisy)


@pytest.mark.parametrize("per_frame_e", [False, True])
def test_host_stream_through_staging_ring(cfg1_ensemble, per_frame_e):
    """300 frames through a 64-frame workspace: 5 chunks, the last partial."""
    import torch

    ens = cfg1_ensemble
    B = 300
    fb = make_frames(ens.n, 0.06, B, seed=5)
    e = np.linspace(0.04, 0.08, B) if per_frame_e else 0.06
    dec = BatchDecoder(ens, 64)
    syn = dec.syndromes(fb.keys)
    res = dec.decode(fb.noisy, syn, e)
    ref = BatchDecoder(ens, B)
    dev = torch.device("cuda:0")
    ed = torch.tensor(np.atleast_1d(e), dtype=torch.float64, device=dev)
    r = ref.decode_device(torch.from_numpy(fb.noisy).to(dev), torch.from_numpy(syn).to(dev), ed)
    torch.cuda.synchronize()
    assert np.array_equal(res.corrected, r[0].cpu().numpy())
    assert np.array_equal(res.converged, r[1].cpu().numpy().astype(bool))
    assert np.array_equal(res.iterations, r[2].cpu().numpy())
    assert np.array_equal(res.mismatches, r[3].cpu().numpy())
    assert res.converged.mean() > 0.9
    # the ring is reused across calls
    res2 = dec.decode(fb.noisy[:130], syn[:130], e[:130] if per_frame_e else e)
    assert np.array_equal(res2.corrected, res.corrected[:130])
    assert np.array_equal(res2.iterations, res.iterations[:130])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    sys.path.insert(0, str(HERE))
    from conftest import _ens, load_golden
    from paper_2001_07979_b200.shard import decode_shard, gather_results, reduce_work_time

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(rank % torch.cuda.device_count())
        ens = _ens("cfg1")
        g = load_golden("golden_cfg1.npz")
        noisy, syn = g["e070_noisy"], g["e070_syn"]
        dec = BatchDecoder(ens, 32, device=torch.cuda.current_device())
        lo, hi, res = decode_shard(dec, noisy, syn, 0.07, world, rank)
        full = gather_results(lo, hi, res, ens.n)
        work, _ = reduce_work_time([float(hi - lo)], [1.0], device=torch.device("cpu"))
        if rank == 0:
            conv = g["e070_converged"]
            ok = (np.array_equal(full["iterations"], g["e070_iterations"])
                  and np.array_equal(full["converged"], conv)
                  and np.array_equal(full["mismatches"], g["e070_mismatches"])
                  and np.array_equal(full["corrected"][conv], g["e070_corrected"][conv]))
            q.put((ok, work))
    finally:
        dist.destroy_process_group()


def test_two_ranks_shard_the_stream_on_the_gpu():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    ok, work = q.get()
    assert ok
    assert work == [32.0]


def test_dropin_decode_per_frame_threads_and_lazy_state(cfg1_ensemble):
    """The reference's measure_throughput pattern: decode() per frame from
    worker threads, with and without a per-thread workspace.  Results equal
    the batched path; a workspace's messages appear on first access and
    equal the eager explicit-kernel readback."""
    from concurrent.futures import ThreadPoolExecutor

    from paper_2001_07979_b200 import BitBlock, DecoderWorkspace, decode
    from paper_2001_07979_b200.decoder import _final_v2c

    ens = cfg1_ensemble
    fb = make_frames(ens.n, 0.07, 24, seed=9)
    dec = BatchDecoder(ens, 24)
    syn = dec.syndromes(fb.keys)
    ref = dec.decode(fb.noisy, syn, 0.07)
    mb = (ens.m + 7) // 8

    def one(k, ws=None):
        return decode(ens, BitBlock(fb.noisy[k], ens.n),
                      [BitBlock(syn[k, l * mb:(l + 1) * mb], ens.m) for l in range(ens.u)], 0.07, workspace=ws)

    with ThreadPoolExecutor(4) as pool:
        got = list(pool.map(one, range(24)))
    for k, r in enumerate(got):
        assert r.converged == bool(ref.converged[k]) and r.iterations_used == int(ref.iterations[k])
        assert np.array_equal(r.corrected.data, ref.corrected[k])
    ws = DecoderWorkspace(ens)
    for k in (0, 5, 11):
        r = one(k, ws)
        assert r.iterations_used == int(ref.iterations[k])
        assert ws._pending is not None                      # nothing read back yet
        c2v, post, v2c = ws.c2v.copy(), ws.posterior.copy(), ws.v2c.copy()
        assert ws._pending is None
        eager = ws._device(ws.config, False)
        eager.decode(fb.noisy[k:k + 1], syn[k:k + 1], 0.07)
        assert np.array_equal(c2v, eager.c2v(0)) and np.array_equal(post, eager.posterior(0))
        assert np.array_equal(v2c, _final_v2c(ws, ws.config, eager))
