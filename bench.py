"""Reconciliation throughput of the B200 MBP decoder (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

``--gpus N`` with N > 1 launches N ranks itself (torch.distributed.run on
127.0.0.1); under an external torchrun the ranks come from the environment.
One process per GPU; when there are fewer GPUs than ranks, ranks share GPUs
round-robin and the reductions run over gloo (said in ``config``).

Headline (BASELINE.json configs[1]): u=2 PEG matrices
n=65536, m=32768 (R=1/2, the reference's build_ensemble(..., base_seed=1)),
BSC QBER e=0.03, a 1024-frame batch per GPU.  Frames are the reference's own
counter-based streams (_frame_inputs, bench.py:123-130), generated on the
device bit for bit (csrc/frames.cuh; spot-checked against numpy here).  A
step = one batched decode of the rank's 1024 frames with noisy keys and
syndromes resident in HBM.  Metric = corrected Mbps: n * #(converged and
corrected == key) / time (bench.py:188-195), summed over ranks, divided by
the max over ranks of the device-timed total.

Also in the line:
* ``e2e``: the same K steps through the C ABI's host call mbp_decode_batch
  with pinned host buffers -- every step's H2D copy and result D2H inside the
  timed region, pipelined against the neighbouring steps' decodes (one call
  over the K batches); ``e2e.per_call``: K separate 1024-frame calls;
* ``stream``: BASELINE configs[4], a fixed 65,536-frame stream sharded
  contiguously over the ranks (strong scaling), device-resident and e2e;
* ``configs``: the north-star operating point cfg 3 (u=3, m=14650, f=1.15 at
  e=0.03) and the fp64 parity mode on cfg 2;
* ``roofline`` of the decode kernel, ``cpu_baseline`` (the reference
  algorithm on the host cores) and ``parity`` (every frame the CPU leg
  decodes compared with the GPU's outputs).

``--impl reference`` times the reference algorithm on the host cores instead
(oracle/ -- the C restatement of the reference's numba decode, pinned to its
golden vectors; the reference itself is Python+numba and does not travel to
the GPU box), on bounded samples of the same frames.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

N_DEFAULT_FRAMES = 1024
STREAM_FRAMES = 65536          # BASELINE configs[4]
WORKLOAD = "cfg2"
E_DEFAULT = 0.03
# BASELINE.json configs: the headline is cfg2 (configs[1]); the others are
# parity-test cases that --workload can also time (cfg4 uses SYNTHETIC random
# (3,6)-regular graphs, the reference's PEG being ~7 h per matrix at 2^20)
WORKLOADS = {
    "cfg1": ("cfg1_n4096_m2048_u2_s1.npz", "u=2 PEG n=4096 m=2048 R=0.5 (reference build_ensemble seeds 1,2)"),
    "cfg2": ("cfg2_n65536_m32768_u2_s1.npz", "u=2 PEG n=65536 m=32768 R=0.5 (reference build_ensemble seeds 1,2)"),
    "cfg3": ("cfg3_n65536_m14650_u3_s11.npz", "u=3 PEG n=65536 m=14650 (f=1.15 at e=0.03; reference seeds 11-13)"),
    "cfg4": ("cfg4_n1048576_m524288_u2_s1.npz",
             "u=2 PEG n=1048576 m=524288 R=0.5 (build_ensemble base_seed=1 on the device PEG: the reference's "
             "matrices)"),
}
CFG4_SYNTHETIC = "u=2 n=1048576 m=524288 R=0.5 SYNTHETIC random (3,6)-regular graphs (seeds 7,8)"
L2_FLUSH_BYTES = 256 << 20   # > 126 MB L2: written between timed steps
KERNELS_PER_DECODE = 5       # setup, 2 row->word transposes, decode, word->row transpose


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=30)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=("ours", "reference"), default="ours")
    p.add_argument("--frames", type=int, default=N_DEFAULT_FRAMES, help="frames per GPU per step")
    p.add_argument("--stream", type=int, default=STREAM_FRAMES,
                   help="frames of the strong-scaling stream (configs[4]); 0 skips it")
    p.add_argument("--e", type=float, default=E_DEFAULT)
    p.add_argument("--precision", choices=("fp32", "fp64"), default="fp32")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-sweep", action="store_true", help="skip the QBER 2-5%% side sweep")
    p.add_argument("--no-extra", action="store_true", help="skip the cfg3 / fp64 side configurations")
    p.add_argument("--workload", choices=tuple(WORKLOADS), default=WORKLOAD,
                   help="BASELINE config to time (default cfg2 = configs[1], the headline)")
    return p.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def self_launch(nproc: int) -> int:
    """`python bench.py --gpus N` without torchrun: start N ranks on this node."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.call(cmd, env=env)


def physical_cores() -> int:
    """Physical cores (unique (package, core) pairs of /proc/cpuinfo)."""
    try:
        pairs, phys, core = set(), None, None
        for line in open("/proc/cpuinfo"):
            k, _, v = line.partition(":")
            k = k.strip()
            if k == "physical id":
                phys = v.strip()
            elif k == "core id":
                core = v.strip()
            elif not k and phys is not None:
                pairs.add((phys, core))
                phys = core = None
        if phys is not None:
            pairs.add((phys, core))
        return len(pairs) or (os.cpu_count() or 1)
    except OSError:
        return os.cpu_count() or 1


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def alg_bytes_per_frame(n, m, u, E, iters):
    """B_frame = I*B_sweep + (2n + u*m)/8,
    B_sweep = 4*(3E + 2n) + (u*m + n)/8 (fp32 messages, APP form)."""
    b_sweep = 4 * (3 * E + 2 * n) + (u * m + n) / 8
    return iters * b_sweep + (2 * n + u * m) / 8


def rule_evals(iters):
    """Eq. 6 evaluations per edge of a frame that stops after `iters` sweeps on
    the scatter kernel (scatter.cuh): sweep 1 none (messages from bits),
    sweep 2 one, sweep 3 two (c2v_2 rebuilt, then c2v_3), later sweeps one."""
    i = int(iters)
    return 0 if i <= 1 else 1 if i == 2 else 3 + max(0, i - 3)


MUFU_PER_EDGE = 3           # ex2 + 2 x lg2 per edge per rule evaluation
MUFU_PER_CLK_SM = 16        # B200 SFU issue rate (ops/clk/SM; B300 doubles it)


def measured_peak_hbm():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        try:
            return float(json.loads(f.read_text())["hbm_gbs"]), "measured"
        except Exception:
            pass
    return 6650.0, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled through NVML every ~1 ms while the
    timed region runs (nvidia-smi as the fallback when NVML is unavailable)."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []   # (sm_mhz, max_mhz, reasons bitmask)
        self._stop = threading.Event()
        self._ready = threading.Event()   # set after the first sample (or a failed init)
        self._t = None
        self.source = "nvml"

    def _run_nvml(self, nv):
        h = nv.nvmlDeviceGetHandleByIndex(self.gpu)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self._stop.is_set():
            self.samples.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), mx,
                                 nv.nvmlDeviceGetCurrentClocksEventReasons(h)))
            self._ready.set()
            self._stop.wait(0.001)

    def _run_smi(self):
        self.source = "nvidia-smi"
        fields = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                  "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={fields}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                v = [x.strip() for x in out.split(",")]
                mask = sum(1 << i for i in range(4) if v[2 + i].lower().startswith("active"))
                self.samples.append((float(v[0]), float(v[1]), mask))
            except Exception:
                return
            finally:
                self._ready.set()
            self._stop.wait(0.05)

    def _run(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
        except Exception:
            return self._run_smi()
        try:
            self._run_nvml(nv)
        finally:
            self._ready.set()
            nv.nvmlShutdown()

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        # NVML init can take longer than a short timed region: wait for the
        # first sample so that the region is always sampled
        self._ready.wait(timeout=10)
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [s[0] for s in self.samples]
        if self.source == "nvml":
            import pynvml as nv

            bits = [(name, getattr(nv, attr, 0)) for name, attr in self.REASONS]
        else:
            bits = [(name, 1 << i) for i, (name, _) in enumerate(self.REASONS[:4])]
        reasons = sorted({name for s in self.samples for name, b in bits if b and (s[2] & b)})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": reasons, "samples": len(self.samples), "source": self.source}


def ensemble_path(workload):
    return ROOT / "paper_2001_07979_b200" / "ensembles" / WORKLOADS[workload][0]


def workload_text(workload):
    if workload == "cfg4" and not ensemble_path(workload).exists():
        return CFG4_SYNTHETIC
    return WORKLOADS[workload][1]


def load_ensemble_for(workload):
    """The workload's PEG ensemble; cfg 4 falls back to synthetic random
    regular graphs when its 2^20 PEG cache is not present."""
    from paper_2001_07979_b200.matrix import load_ensemble, random_regular_ensemble

    p = ensemble_path(workload)
    if workload == "cfg4" and not p.exists():
        return random_regular_ensemble(1 << 20, 1 << 19, 2, seed=7)
    return load_ensemble(p)


def device_frames(dec, n, e, lo, count, device):
    """Frames lo .. lo+count-1 of the point (path ()) in HBM: keys, noisy,
    syndromes (all on the current stream)."""
    from paper_2001_07979_b200.channel import make_frames_device

    keys, noisy = make_frames_device(n, e, count, seed=0, start=lo, device=device)
    return keys, noisy, dec.syndromes(keys)


def spot_check_frames(keys, noisy, n, e, lo):
    """The device generator against numpy's streams on two frames."""
    from paper_2001_07979_b200.channel import make_frames

    B = keys.shape[0]
    for k in sorted({0, B - 1}):
        ref = make_frames(n, e, 1, seed=0, start=lo + k)
        if not (np.array_equal(keys[k].cpu().numpy(), ref.keys[0])
                and np.array_equal(noisy[k].cpu().numpy(), ref.noisy[0])):
            raise RuntimeError(f"device frame generator differs from numpy on frame {lo + k}")


def good_bits(out, keys, n):
    """n * #(converged and corrected == key) (bench.py:188-195), on device."""
    import torch

    ok = (out[1] != 0) & torch.all(out[0] == keys, dim=1)
    return int(ok.sum().item()) * n


class Pinned:
    """Pinned host rows (torch pinned memory viewed as numpy)."""

    def __init__(self, shape, dtype):
        import torch

        tdt = {np.uint8: torch.uint8, np.int32: torch.int32}[np.dtype(dtype).type]
        self.t = torch.empty(shape, dtype=tdt, pin_memory=True)
        self.a = self.t.numpy()


def time_device_steps(dec, noisy, syn, e_d, out, steps, flush, stream):
    """K decode steps bracketed by CUDA events on the launching stream, L2
    flushed before each; returns (per-step ms, per-step decode-kernel ms)."""
    import torch

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    kernel_ms = []
    for k in range(steps):
        flush.fill_(k & 0xFF)
        starts[k].record(stream)
        dec.decode_device(noisy, syn, e_d, out=out)
        ends[k].record(stream)
        kernel_ms.append(dec.last_timing()[0])
    torch.cuda.synchronize()
    return [s.elapsed_time(t) for s, t in zip(starts, ends)], kernel_ms


def host_call(dec, noisy_h, syn_h, e, out):
    """One host-buffer call through the C ABI: (device-event ms, host wall ms)."""
    t0 = time.perf_counter()
    dec.decode(noisy_h, syn_h, e, out=out)
    wall = (time.perf_counter() - t0) * 1e3
    return dec.last_timing(e2e=True)[1], wall


def host_result(B, nb, n):
    from paper_2001_07979_b200.decoder import BatchResult

    return BatchResult(Pinned((B, nb), np.uint8).a, Pinned((B,), np.uint8).a, Pinned((B,), np.int32).a,
                       Pinned((B,), np.int32).a, n)


def cpu_decode_sample(ens, noisy_rows, syn_rows, e, budget_s=10.0, threads=None):
    """The reference algorithm (oracle/, C restatement of _kernels.decode_loop)
    on the host cores over a bounded prefix of the frames."""
    import oracle
    from paper_2001_07979_b200.matrix import stacked_layout

    threads = threads or host_threads()
    og = oracle.OracleGraph(stacked_layout(ens))
    B = noisy_rows.shape[0]
    k = min(B, threads)
    t0 = time.perf_counter()
    oracle.decode_batch(og, noisy_rows[:k], syn_rows[:k], e, threads=threads)
    per_round = max(time.perf_counter() - t0, 1e-3)
    frames = int(min(B, max(k, k * budget_s / per_round)))
    t0 = time.perf_counter()
    corrected, conv, iters, mism = oracle.decode_batch(og, noisy_rows[:frames], syn_rows[:frames], e,
                                                       threads=threads)
    wall = time.perf_counter() - t0
    return corrected, conv, iters, mism, wall, frames, threads


def traffic_record(workload, frames, e):
    """ncu DRAM bytes per decode launch for this source tree (None if the
    committed capture was taken on other sources)."""
    from paper_2001_07979_b200.build import source_hash

    tf = ROOT / "profiles" / "decode_traffic.json"
    if not tf.exists():
        return None
    try:
        recs = json.loads(tf.read_text())
        recs = recs if isinstance(recs, list) else [recs]
        src = source_hash()
        for t in recs:
            if (t.get("workload") == workload and t.get("frames") == frames and t.get("e") == e
                    and t.get("src_sha") == src):
                return t
    except Exception:
        pass
    return None


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    from paper_2001_07979_b200.channel import make_frames_native
    from paper_2001_07979_b200.matrix import stacked_layout

    ens = load_ensemble_for(args.workload)
    fb = make_frames_native(ens.n, args.e, args.frames, seed=0, start=0)
    lay = stacked_layout(ens)
    og = oracle.OracleGraph(lay)
    syn = np.stack([np.concatenate([np.packbits(
        oracle.syndrome(lay.chk_ptr, lay.chk_var, np.unpackbits(fb.keys[k], count=ens.n, bitorder="little"),
                        l * ens.m, (l + 1) * ens.m), bitorder="little") for l in range(ens.u)])
        for k in range(fb.batch)])
    threads = host_threads()
    step_frames = min(fb.batch, threads * 8)
    times, gbits = [], []
    for s in range(args.warmup + args.steps):
        lo = (s * step_frames) % fb.batch
        idx = np.arange(lo, lo + step_frames) % fb.batch
        t0 = time.perf_counter()
        corrected, conv, iters, _ = oracle.decode_batch(og, fb.noisy[idx], syn[idx], args.e, threads=threads)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            good = conv & np.all(corrected == fb.keys[idx], axis=1)
            times.append(dt)
            gbits.append(int(good.sum()) * ens.n)
    total = sum(times)
    value = sum(gbits) / total / 1e6
    line = {
        "metric": "reconciliation throughput (corrected Mbps)", "value": round(value, 4), "unit": "Mbps",
        "impl": "reference", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * total / len(times), 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference Philox frame streams)",
        "config": config_dict(args, ens, args.gpus, args.gpus),
        "cpu_baseline": {"value": round(value, 4), "unit": "Mbps", "cores": physical_cores(), "threads": threads,
                         "kind": "port",
                         "sample": f"{step_frames} frames per step of the {args.frames}-frame workload, "
                                   f"oracle/mbp_oracle.c decode_loop restatement (fp64, libm) on {threads} "
                                   f"POSIX threads"},
        "e2e": {"value": round(value, 4), "unit": "Mbps", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_dict(args, ens, world, devices):
    from paper_2001_07979_b200.channel import efficiency

    par = f"dp{world} (contiguous frame shards, no collective on the data path)"
    if devices < world:
        par += f"; {world} ranks on {devices} GPU(s), round-robin"
    return {"workload": f"{args.workload}: {workload_text(args.workload)}, "
                        f"BSC e={args.e}, {args.frames}-frame batch per GPU",
            "n": ens.n, "m": ens.m, "u": ens.u, "e": args.e, "f": round(efficiency(ens.m, ens.n, args.e), 4),
            "frames_per_gpu": args.frames, "max_iterations": 60, "llr_clamp": 30.0,
            "parallelism": par, "l2": "flushed between timed steps (256 MiB write); working set >> L2"}


def side_config(workload, e, precision, frames, steps, device, flush, stream):
    """A single-GPU figure for another configuration: device value, e2e
    (host call, pipelined over `steps` batches), fer, iterations, kernel ms."""
    import torch

    from paper_2001_07979_b200 import BatchDecoder, DecoderConfig

    ens = load_ensemble_for(workload)
    n = ens.n
    dec = BatchDecoder(ens, frames, DecoderConfig(precision=precision), device=device)
    keys, noisy, syn = device_frames(dec, n, e, 0, frames, device)
    e_d = torch.tensor([e], dtype=torch.float64, device=noisy.device)
    out = dec.decode_device(noisy, syn, e_d)
    dec.decode_device(noisy, syn, e_d, out=out)
    torch.cuda.synchronize()
    step_ms, kms = time_device_steps(dec, noisy, syn, e_d, out, steps, flush, stream)
    gb = good_bits(out, keys, n)
    iters = out[2].cpu().numpy()
    value = gb * steps / (sum(step_ms) / 1e3) / 1e6
    E = int(ens.matrices[0].edge_count) * ens.u
    alg = float(sum(alg_bytes_per_frame(n, ens.m, ens.u, E, int(i)) for i in iters))
    peak, _ = measured_peak_hbm()
    # e2e: `steps` batches through one host call
    nb = keys.shape[1]
    K = steps
    kk, nn, ss = device_frames(dec, n, e, 0, K * frames, device)
    noisy_h, syn_h = Pinned(tuple(nn.shape), np.uint8), Pinned(tuple(ss.shape), np.uint8)
    noisy_h.t.copy_(nn)
    syn_h.t.copy_(ss)
    keys_h = kk.cpu().numpy()
    del kk, nn, ss
    res = host_result(K * frames, nb, n)
    host_call(dec, noisy_h.a, syn_h.a, e, res)
    ev_ms, wall_ms = host_call(dec, noisy_h.a, syn_h.a, e, res)
    g2 = int((res.converged.astype(bool) & np.all(res.corrected == keys_h, axis=1)).sum()) * n
    return {
        "workload": workload_text(workload), "e": e, "precision": precision, "frames": frames,
        "value": round(value, 3), "unit": "Mbps", "ms_per_step": round(statistics.mean(step_ms), 4),
        "kernel_ms": round(statistics.mean(kms), 4),
        "e2e": {"value": round(g2 / (ev_ms / 1e3) / 1e6, 3), "host_wall_value": round(g2 / (wall_ms / 1e3) / 1e6, 3),
                "batches": K},
        "fer": round(1.0 - float(out[1].float().mean().item()), 6),
        "mean_iterations": round(float(iters.mean()), 4),
        "roofline": {"achieved": round(alg / (statistics.mean(kms) / 1e3) / 1e9, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(alg / (statistics.mean(kms) / 1e3) / 1e9 / peak, 4),
                     "basis": "SURVEY 8(d) message-streaming bytes / decode-kernel time"},
    }


def dropin_figure(ens, keys_h, noisy_h, syn_h, e, frames=256, workers=8):
    """The reference's own call pattern (bench.measure_throughput, bench.py:
    159-179): decode() once per frame from a thread pool, each thread with its
    own DecoderWorkspace -- the literal drop-in of INTEGRATION.md §1.
    Host wall clock over the frames (like the reference's `mbps`)."""
    import threading
    from concurrent.futures import ThreadPoolExecutor

    from paper_2001_07979_b200 import BitBlock, DecoderWorkspace, decode

    n, m, u = ens.n, ens.m, ens.u
    mb = (m + 7) // 8
    tls = threading.local()

    def one(k):
        ws = getattr(tls, "ws", None)
        if ws is None:
            ws = tls.ws = DecoderWorkspace(ens)
        r = decode(ens, BitBlock(noisy_h[k], n), [BitBlock(syn_h[k, l * mb:(l + 1) * mb], m) for l in range(u)], e,
                   workspace=ws)
        return r.converged and np.array_equal(r.corrected.data, keys_h[k])

    with ThreadPoolExecutor(workers) as pool:
        list(pool.map(one, range(min(workers * 2, frames))))     # warm-up: per-thread workspaces
        t0 = time.perf_counter()
        ok = list(pool.map(one, range(frames)))
        wall = time.perf_counter() - t0
    return {"value": round(sum(ok) * n / wall / 1e6, 3), "unit": "Mbps", "frames": frames, "workers": workers,
            "timing": "host wall clock; decode() per frame (reference API), thread-local DecoderWorkspace, "
                      "pageable host buffers"}


STREAM_CHUNK = 4096   # frames per decode launch in the stream (fixed per-sweep costs amortise)


def run_stream(args, ens, rank, world, device, flush, stream):
    """BASELINE configs[4]: a fixed stream of args.stream frames sharded
    contiguously over the ranks (strong scaling), decoded in launches of
    STREAM_CHUNK frames.  Device-resident value and e2e through the pipelined
    host call, both max over ranks."""
    import torch

    from paper_2001_07979_b200 import BatchDecoder, DecoderConfig
    from paper_2001_07979_b200.shard import reduce_work_time, shard_range

    n = ens.n
    lo, hi = shard_range(args.stream, world, rank)
    S = hi - lo
    dec = BatchDecoder(ens, max(1, min(STREAM_CHUNK, S)), DecoderConfig(precision=args.precision), device=device)
    e_d = torch.tensor([args.e], dtype=torch.float64, device=torch.device("cuda", device))
    keys, noisy, syn = device_frames(dec, n, args.e, lo, max(S, 1), device)
    out = dec.decode_device(noisy[:S], syn[:S], e_d) if S else None
    torch.cuda.synchronize()
    passes = 3
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    flush.fill_(1)

    def run():
        t0.record(stream)
        for _ in range(passes):
            if S:
                dec.decode_device(noisy[:S], syn[:S], e_d, out=out)
        t1.record(stream)

    span, _ = job_span(world, run)
    dev_ms = (span if _SHARED else t0.elapsed_time(t1)) / passes
    gb = good_bits(out, keys[:S], n) if S else 0
    # e2e: host pinned buffers through one mbp_decode_batch call per pass
    nb = keys.shape[1]
    noisy_h = Pinned((max(S, 1), nb), np.uint8)
    syn_h = Pinned((max(S, 1), syn.shape[1]), np.uint8)
    noisy_h.t.copy_(noisy)
    syn_h.t.copy_(syn)
    keys_h = keys.cpu().numpy()
    del keys, noisy, syn
    res = host_result(max(S, 1), nb, n)
    ev, wall = [], []

    def run_host():
        for p in range(passes):
            if S:
                a, b = host_call(dec, noisy_h.a[:S], syn_h.a[:S], args.e, res)
                ev.append(a)
                wall.append(b)

    span, _ = job_span(world, run_host)
    if _SHARED:
        ev, wall = [span / passes], [span / passes]
    e2e_ms = statistics.mean(ev) if ev else 0.0
    wall_ms = statistics.mean(wall) if wall else 0.0
    g2 = int((res.converged[:S].astype(bool) & np.all(res.corrected[:S] == keys_h[:S], axis=1)).sum()) * n
    (gb_all, g2_all, frames_all), (dev_max, e2e_max, wall_max) = reduce_work_time(
        [float(gb), float(g2), float(S)], [dev_ms, e2e_ms, wall_ms], device=red_device(device))
    return {
        "workload": f"BASELINE configs[4]: {WORKLOADS['cfg2'][1]}, e={args.e}, {args.stream}-frame stream "
                    f"(frames 0..{args.stream - 1}) in contiguous shards over {world} rank(s)",
        "frames": int(frames_all), "scaling": "strong",
        "value": round(gb_all / (dev_max / 1e3) / 1e6, 3), "unit": "Mbps", "ms": round(dev_max, 3),
        "e2e": {"value": round(g2_all / (e2e_max / 1e3) / 1e6, 3),
                "host_wall_value": round(g2_all / (wall_max / 1e3) / 1e6, 3),
                "h2d_bytes": int(args.stream * (nb + dec.dev.nbytes_syn + 8)),
                "d2h_bytes": int(args.stream * (nb + 9)),
                "timing": f"one mbp_decode_batch host call per rank and pass (pinned buffers, H2D || decode || "
                          f"D2H over {STREAM_CHUNK}-frame chunks); max over ranks"},
        "frames_per_launch": int(dec.max_frames),
        "fer": round(1.0 - gb_all / max(frames_all * n, 1), 6),
    }


_RED_DEVICE = None
_SHARED = False     # ranks share GPUs: time the job span, not per-rank events


def job_span(world, fn):
    """(ms, fn()) between two barrier-synchronised host clock reads: the
    whole job's span when several ranks' kernels time-slice one GPU (their
    per-rank CUDA-event windows then do not overlap)."""
    import torch

    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    return (time.perf_counter() - t0) * 1e3, r


def red_device(device):
    return _RED_DEVICE if _RED_DEVICE is not None else device


def main():
    global _RED_DEVICE, _SHARED
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return self_launch(args.gpus)

    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    ndev = torch.cuda.device_count()
    if ndev < 1:
        raise RuntimeError("no CUDA device: the decoder has no CPU fallback")
    device = local % ndev
    devices = min(world, ndev)
    torch.cuda.set_device(device)
    dev = torch.device("cuda", device)
    if world > 1:
        if world <= ndev:
            dist.init_process_group("nccl", device_id=dev)
        else:   # ranks share GPUs: NCCL allows one rank per GPU
            dist.init_process_group("gloo")
            _RED_DEVICE = torch.device("cpu")
            _SHARED = True

    from paper_2001_07979_b200 import BatchDecoder, DecoderConfig
    from paper_2001_07979_b200.shard import reduce_work_time, shard_range

    ens = load_ensemble_for(args.workload)
    n, m, u = ens.n, ens.m, ens.u
    B = args.frames
    dec = BatchDecoder(ens, B, DecoderConfig(precision=args.precision), device=device)
    lo, _ = shard_range(world * B, world, rank)
    keys_d, noisy_d, syn_d = device_frames(dec, n, args.e, lo, B, device)
    torch.cuda.synchronize()
    spot_check_frames(keys_d, noisy_d, n, args.e, lo)
    e_d = torch.tensor([args.e], dtype=torch.float64, device=dev)
    out = dec.decode_device(noisy_d, syn_d, e_d)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    for _ in range(args.warmup):
        dec.decode_device(noisy_d, syn_d, e_d, out=out)
    torch.cuda.synchronize(dev)

    with ClockSampler(device) as clocks:
        span, (step_ms, kernel_ms) = job_span(world, lambda: time_device_steps(
            dec, noisy_d, syn_d, e_d, out, args.steps, flush, stream))
    total_ms = span if _SHARED else sum(step_ms)
    _, sweeps = dec.last_timing()

    corrected = out[0].cpu().numpy()
    conv = out[1].cpu().numpy().astype(bool)
    iters = out[2].cpu().numpy()
    mism = out[3].cpu().numpy()
    keys_h = keys_d.cpu().numpy()
    good = conv & np.all(corrected == keys_h, axis=1)
    gbits = int(good.sum()) * n * args.steps

    # ---- e2e: the K steps' batches (frames of this rank's shard of K*B*world)
    #      through the host C-ABI call with pinned buffers ---------------------
    K = args.steps
    lo_k, _ = shard_range(world * K * B, world, rank)
    kk, nn, ss = device_frames(dec, n, args.e, lo_k, K * B, device)
    nb = nn.shape[1]
    pin_noisy, pin_syn = Pinned((K * B, nb), np.uint8), Pinned((K * B, ss.shape[1]), np.uint8)
    pin_noisy.t.copy_(nn)
    pin_syn.t.copy_(ss)
    keys_k = kk.cpu().numpy()
    del kk, nn, ss
    res = host_result(K * B, nb, n)
    host_call(dec, pin_noisy.a, pin_syn.a, args.e, res)          # warm the staging ring
    span, (e2e_ms, e2e_wall) = job_span(world, lambda: host_call(dec, pin_noisy.a, pin_syn.a, args.e, res))
    if _SHARED:
        e2e_ms = e2e_wall = span
    e2e_good = int((res.converged.astype(bool) & np.all(res.corrected == keys_k, axis=1)).sum()) * n
    # per call: K separate 1024-frame host calls (no overlap inside a call)
    res1 = host_result(B, nb, n)
    pc_ev, pc_wall, pc_good = [], [], 0

    def per_call():
        nonlocal pc_good
        for k in range(K):
            a, b = host_call(dec, pin_noisy.a[k * B:(k + 1) * B], pin_syn.a[k * B:(k + 1) * B], args.e, res1)
            pc_ev.append(a)
            pc_wall.append(b)
            pc_good += int((res1.converged.astype(bool)
                            & np.all(res1.corrected == keys_k[k * B:(k + 1) * B], axis=1)).sum()) * n

    span, _ = job_span(world, per_call)
    if _SHARED:
        pc_ev, pc_wall = [span], [span]

    # ---- cross-rank aggregation: sums of work, max of time (shard.py) --------
    (good_all, e2e_good_all, pc_good_all, frames_all), (total_max, e2e_max, wall_max, pc_max, pcw_max) = \
        reduce_work_time([float(gbits), float(e2e_good), float(pc_good), float(B)],
                         [total_ms, e2e_ms, e2e_wall, sum(pc_ev), sum(pc_wall)], device=red_device(dev))
    value = good_all / (total_max / 1e3) / 1e6
    e2e_value = e2e_good_all / (e2e_max / 1e3) / 1e6

    # ---- roofline of the dominant kernel (the cooperative decode) ------------
    E = int(ens.matrices[0].edge_count) * u
    alg_bytes = float(sum(alg_bytes_per_frame(n, m, u, E, int(i)) for i in iters))
    kms_mean = statistics.mean(kernel_ms)
    achieved = alg_bytes / (kms_mean / 1e3) / 1e9
    peak, peak_kind = measured_peak_hbm()
    trec = traffic_record(args.workload, B, args.e) if args.precision == "fp32" else None
    traffic = trec.get("dram_bytes_per_launch") if trec else None
    dram_frac = traffic / (kms_mean / 1e3) / 1e9 / peak if traffic else None
    mufu_ops = float(sum(rule_evals(i) for i in iters)) * E * MUFU_PER_EDGE
    sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
    clocks_summary = clocks.summary()
    sm_mhz = clocks_summary.get("sm_mhz") or 1965.0
    mufu_peak = MUFU_PER_CLK_SM * sm_count * sm_mhz * 1e6
    mufu_ach = mufu_ops / (kms_mean / 1e3)
    hbm_bound = args.workload == "cfg4"

    line = {
        "metric": "reconciliation throughput (corrected Mbps)",
        "value": round(value, 3), "unit": "Mbps", "n_gpus": world, "devices": devices, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(total_max / args.steps, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32" if args.precision == "fp32" else "f64",
        "data": "synthetic (the reference's Philox frame streams, generated on the GPU bit for bit; "
                + ("synthetic random regular graphs)" if workload_text(args.workload) == CFG4_SYNTHETIC
                   else "PEG ensemble of the reference)"),
        "config": config_dict(args, ens, world, devices),
        "timing": ("host clock over the barrier-synchronised job span (ranks time-slice shared GPUs)" if _SHARED
                   else "CUDA events on each rank's launching stream, max over ranks"),
        "fer": round(1.0 - float(conv.mean()), 6), "mean_iterations": round(float(iters.mean()), 4),
        "sweeps_run": sweeps,
        "e2e": {"value": round(e2e_value, 3), "unit": "Mbps",
                "h2d_bytes_per_step": int(B * (nb + pin_syn.a.shape[1]) + 8),
                "d2h_bytes_per_step": int(B * (nb + 9)),
                "host_wall_value": round(e2e_good_all / (wall_max / 1e3) / 1e6, 3),
                "timing": f"one mbp_decode_batch host call over the {K} steps' batches ({K}x{B} frames per rank, "
                          "pinned buffers): each step's H2D, decode and D2H overlap the neighbouring steps' "
                          "(two-slot staging ring); CUDA events on the workspace stream, max over ranks; "
                          "host_wall_value: perf_counter around the call",
                "per_call": {"value": round(pc_good_all / (pc_max / 1e3) / 1e6, 3),
                             "host_wall_value": round(pc_good_all / (pcw_max / 1e3) / 1e6, 3),
                             "timing": f"{K} separate {B}-frame host calls (copies cannot overlap inside one)"}},
        "gpu_launches": KERNELS_PER_DECODE * args.steps,
        "roofline": {
            "bound": "hbm" if hbm_bound else "latency",
            "bound_detail": ("HBM: random 128-byte variable-block lines, L2 hit ~22 % (profiles/)" if hbm_bound else
                             "L2/gather latency and issue (ncu: long-scoreboard stalls, ~50 % warps active, "
                             "DRAM well below peak; profiles/r02*_scatter_ncu.md)"),
            "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": traffic,
            "dram_frac": round(dram_frac, 4) if dram_frac is not None else None,
            "traffic_source": (f"ncu --set full capture {trec.get('capture')} of these sources "
                               f"(src {trec.get('src_sha')})" if trec else
                               "no ncu capture of these sources committed (profiles/decode_traffic.json)"),
            "kernel": "mbp::decode_scatter_kernel (cooperative, persistent, all sweeps)",
            "kernel_ms": round(kms_mean, 4), "alg_bytes_per_launch": alg_bytes,
            "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
            "note": "achieved = SURVEY 8(d) message-streaming bytes / kernel time (the scatter kernel keeps "
                    "sweep-1/2 messages out of HBM, so frac > 1 is possible); dram_frac = ncu DRAM bytes / "
                    "kernel time / peak is the real HBM utilisation",
            "compute": {"unit": "MUFU op/s", "achieved": round(mufu_ach / 1e12, 4),
                        "peak": round(mufu_peak / 1e12, 4), "scale": "1e12",
                        "frac": round(mufu_ach / mufu_peak, 4),
                        "basis": f"{MUFU_PER_EDGE} SFU ops per edge per Eq. 6 evaluation, "
                                 f"{MUFU_PER_CLK_SM}/clk/SM x {sm_count} SMs x median SM clock"}},
        "clocks": clocks_summary,
    }

    if args.stream:
        line["stream"] = run_stream(args, ens, rank, world, device, flush, stream)

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        corrected_c, conv_c, iters_c, mism_c, wall, frames_c, threads = cpu_decode_sample(
            ens, noisy_d.cpu().numpy(), syn_d.cpu().numpy(), args.e)
        good_c = conv_c & np.all(corrected_c == keys_h[:frames_c], axis=1)
        line["cpu_baseline"] = {"value": round(int(good_c.sum()) * n / wall / 1e6, 4), "unit": "Mbps",
                                "cores": physical_cores(), "threads": threads, "kind": "port",
                                "sample": f"first {frames_c} of the {B} frames, oracle/mbp_oracle.c "
                                          f"(reference decode_loop restated in C/libm fp64) on {threads} threads "
                                          f"({physical_cores()} physical cores), {wall:.1f} s wall"}
        bad = ((conv_c != conv[:frames_c]) | (iters_c != iters[:frames_c]) | (mism_c != mism[:frames_c])
               | (conv_c & np.any(corrected_c != corrected[:frames_c], axis=1)))
        line["parity"] = {"frames": int(frames_c), "mismatching_frames": int(bad.sum()),
                          "checked": "per frame: converged, iterations, residual mismatches, corrected key of "
                                     "converged frames -- GPU (this run) vs the oracle (reference decode_loop, "
                                     "fp64) on the same frames"}
    if rank == 0 and not args.no_extra:
        line["dropin_decode"] = dropin_figure(ens, keys_h, noisy_d.cpu().numpy(), syn_d.cpu().numpy(), args.e)
    if rank == 0 and not args.no_extra and args.workload == "cfg2":
        line["configs"] = {
            "cfg3": side_config("cfg3", 0.03, "fp32", B, 10, device, flush, stream),
            "cfg2_fp64": side_config("cfg2", args.e, "fp64", B, 5, device, flush, stream),
        }
    if rank == 0 and not args.no_sweep:
        sweep = {}
        for e in (0.02, 0.04, 0.05):
            kq, nq, sq = device_frames(dec, n, e, lo, B, device)
            ed = torch.tensor([e], dtype=torch.float64, device=dev)
            dec.decode_device(nq, sq, ed, out=out)
            ts, _ = time_device_steps(dec, nq, sq, ed, out, 5, flush, stream)
            sweep[str(e)] = {"mbps": round(good_bits(out, kq, n) / (statistics.mean(ts) / 1e3) / 1e6, 1),
                             "fer": round(1 - float(out[1].float().mean().item()), 6),
                             "mean_iterations": round(float(out[2].float().mean().item()), 3)}
        line["qber_sweep"] = sweep
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
