"""Reconciliation throughput of the B200 MBP decoder (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU)

Workload (BASELINE.json configs[1]): u=2 PEG matrices
n=65536, m=32768 (R=0.5, the reference's build_ensemble(..., base_seed=1)),
BSC QBER e=0.03, a 1024-frame batch per GPU; frames are the reference's own
counter-based streams (_frame_inputs, bench.py:123-130) for frame indices
rank*1024 + i.  A step = one batched decode of the rank's 1024 frames with
noisy keys and syndromes already resident in HBM.  Metric = corrected Mbps:
n * #(converged and corrected == key) / time (bench.py:188-195), summed over
ranks, divided by the max over ranks of the device-timed step total.

``--impl reference`` times the reference algorithm on the host cores instead
(oracle/ -- the C restatement of the reference's numba decode, pinned to its
golden vectors; the reference itself is Python+numba and does not travel to
the GPU box), on bounded samples of the same frames.
"""

from __future__ import annotations

import argparse
import json
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

N_DEFAULT_FRAMES = 1024
WORKLOAD = "cfg2"
E_DEFAULT = 0.03
# BASELINE.json configs: the headline is cfg2 (configs[1]); the others are
# parity-test cases that --workload can also time (cfg4 uses SYNTHETIC random
# (3,6)-regular graphs, the reference's PEG being ~7 h per matrix at 2^20)
WORKLOADS = {
    "cfg1": ("cfg1_n4096_m2048_u2_s1.npz", "u=2 PEG n=4096 m=2048 R=0.5 (reference build_ensemble seeds 1,2)"),
    "cfg2": ("cfg2_n65536_m32768_u2_s1.npz", "u=2 PEG n=65536 m=32768 R=0.5 (reference build_ensemble seeds 1,2)"),
    "cfg3": ("cfg3_n65536_m14650_u3_s11.npz", "u=3 PEG n=65536 m=14650 (f=1.15 at e=0.03; reference seeds 11-13)"),
    "cfg4": (None, "u=2 n=1048576 m=524288 R=0.5 SYNTHETIC random (3,6)-regular graphs (seeds 7,8)"),
}
L2_FLUSH_BYTES = 256 << 20   # > 126 MB L2: written between timed steps


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=30)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=("ours", "reference"), default="ours")
    p.add_argument("--frames", type=int, default=N_DEFAULT_FRAMES, help="frames per GPU per step")
    p.add_argument("--e", type=float, default=E_DEFAULT)
    p.add_argument("--precision", choices=("fp32", "fp64"), default="fp32")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-sweep", action="store_true", help="skip the QBER 2-5%% side sweep")
    p.add_argument("--workload", choices=tuple(WORKLOADS), default=WORKLOAD,
                   help="BASELINE config to time (default cfg2 = configs[1], the headline)")
    return p.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


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
        self._t = None
        self.source = "nvml"

    def _run_nvml(self, nv):
        h = nv.nvmlDeviceGetHandleByIndex(self.gpu)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self._stop.is_set():
            self.samples.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), mx,
                                 nv.nvmlDeviceGetCurrentClocksEventReasons(h)))
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
            nv.nvmlShutdown()

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        time.sleep(0.005)   # first sample before the timed region
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


def load_workload(rank, frames, e, world=1, workload=WORKLOAD):
    """Rank's shard of the frame stream: frames [rank*B, (rank+1)*B) of the
    reference's counter-based streams (shard.shard_range over world*B frames,
    weak scaling: B frames per GPU)."""
    from paper_2001_07979_b200.channel import make_frames
    from paper_2001_07979_b200.matrix import load_ensemble, random_regular_ensemble
    from paper_2001_07979_b200.shard import shard_range

    fname = WORKLOADS[workload][0]
    ens = (load_ensemble(ROOT / "paper_2001_07979_b200" / "ensembles" / fname) if fname
           else random_regular_ensemble(1 << 20, 1 << 19, 2, seed=7))
    lo, hi = shard_range(world * frames, world, rank)
    fb = make_frames(ens.n, e, hi - lo, seed=0, start=lo)
    return ens, fb


def cpu_decode_sample(ens, noisy_rows, syn_rows, e, budget_s=10.0, threads=None):
    """The reference algorithm (oracle/, C restatement of _kernels.decode_loop)
    on the host cores over a bounded prefix of the frames; returns (Mbps, info)."""
    import oracle
    from paper_2001_07979_b200.matrix import stacked_layout

    threads = threads or os.cpu_count() or 1
    og = oracle.OracleGraph(stacked_layout(ens))
    # calibrate on one frame per thread, then size the sample to ~budget_s
    B = noisy_rows.shape[0]
    k = min(B, threads)
    t0 = time.perf_counter()
    oracle.decode_batch(og, noisy_rows[:k], syn_rows[:k], e, threads=threads)
    per_round = max(time.perf_counter() - t0, 1e-3)
    frames = int(min(B, max(k, k * budget_s / per_round)))
    t0 = time.perf_counter()
    corrected, conv, iters, _ = oracle.decode_batch(og, noisy_rows[:frames], syn_rows[:frames], e, threads=threads)
    wall = time.perf_counter() - t0
    return corrected, conv, iters, wall, frames, threads


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    ens, fb = load_workload(0, args.frames, args.e, 1, args.workload)
    import oracle
    from paper_2001_07979_b200.matrix import stacked_layout

    lay = stacked_layout(ens)
    og = oracle.OracleGraph(lay)
    syn = np.stack([np.concatenate([np.packbits(
        oracle.syndrome(lay.chk_ptr, lay.chk_var, np.unpackbits(fb.keys[k], count=ens.n, bitorder="little"),
                        l * ens.m, (l + 1) * ens.m), bitorder="little") for l in range(ens.u)])
        for k in range(fb.batch)])
    threads = os.cpu_count() or 1
    step_frames = min(fb.batch, threads * 8)
    times, good_bits = [], []
    for s in range(args.warmup + args.steps):
        lo = (s * step_frames) % fb.batch
        idx = np.arange(lo, lo + step_frames) % fb.batch
        t0 = time.perf_counter()
        corrected, conv, iters, _ = oracle.decode_batch(og, fb.noisy[idx], syn[idx], args.e, threads=threads)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            good = conv & np.all(corrected == fb.keys[idx], axis=1)
            times.append(dt)
            good_bits.append(int(good.sum()) * ens.n)
    total = sum(times)
    value = sum(good_bits) / total / 1e6
    line = {
        "metric": "reconciliation throughput (corrected Mbps)", "value": round(value, 4), "unit": "Mbps",
        "impl": "reference", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * total / len(times), 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference Philox frame streams)",
        "config": config_dict(args, ens),
        "cpu_baseline": {"value": round(value, 4), "unit": "Mbps", "cores": threads, "kind": "port",
                         "sample": f"{step_frames} frames per step of the {args.frames}-frame workload, "
                                   f"oracle/mbp_oracle.c decode_loop restatement on {threads} POSIX threads"},
        "e2e": {"value": round(value, 4), "unit": "Mbps", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_dict(args, ens):
    from paper_2001_07979_b200.channel import efficiency

    return {"workload": f"{args.workload}: {WORKLOADS[args.workload][1]}, "
                        f"BSC e={args.e}, {args.frames}-frame batch per GPU",
            "n": ens.n, "m": ens.m, "u": ens.u, "e": args.e, "f": round(efficiency(ens.m, ens.n, args.e), 4),
            "frames_per_gpu": args.frames, "max_iterations": 60, "llr_clamp": 30.0,
            "precision": args.precision, "parallelism": f"dp{args.gpus} (frame shards, no collective)",
            "l2": "flushed between timed steps (256 MiB write); working set >> L2"}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)

    from paper_2001_07979_b200 import BatchDecoder, DecoderConfig

    ens, fb = load_workload(rank, args.frames, args.e, world, args.workload)
    n, m, u = ens.n, ens.m, ens.u
    B = fb.batch
    dec = BatchDecoder(ens, B, DecoderConfig(precision=args.precision), device=local)
    keys_d = torch.from_numpy(fb.keys).to(dev)
    noisy_d = torch.from_numpy(fb.noisy).to(dev)
    syn_d = dec.syndromes(keys_d)
    e_d = torch.tensor([args.e], dtype=torch.float64, device=dev)
    out = (torch.empty_like(noisy_d), torch.empty(B, dtype=torch.uint8, device=dev),
           torch.empty(B, dtype=torch.int32, device=dev), torch.empty(B, dtype=torch.int32, device=dev))
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    for _ in range(args.warmup):
        dec.decode_device(noisy_d, syn_d, e_d, out=out)
    torch.cuda.synchronize(dev)

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    kernel_ms = []
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clocks:
        for k in range(args.steps):
            flush.fill_(k & 0xFF)
            starts[k].record(stream)
            dec.decode_device(noisy_d, syn_d, e_d, out=out)
            ends[k].record(stream)
            kms, _sw = dec.last_timing()
            kernel_ms.append(kms)
        torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = sum(step_ms)
    _, sweeps = dec.last_timing()

    corrected = out[0].cpu().numpy()
    conv = out[1].cpu().numpy().astype(bool)
    iters = out[2].cpu().numpy()
    good = conv & np.all(corrected == fb.keys, axis=1)
    good_bits = int(good.sum()) * n * args.steps

    # ---- e2e: host pinned buffers through the C-ABI host call --------------
    from paper_2001_07979_b200.decoder import BatchResult

    pin_noisy = torch.from_numpy(fb.noisy).pin_memory().numpy()
    pin_syn = syn_d.cpu().pin_memory().numpy()
    # caller-owned pinned result buffers (BatchDecoder.decode's `out`)
    pin_out = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
    out_host = BatchResult(pin_out(np.empty_like(fb.noisy)), pin_out(np.empty(B, dtype=np.uint8)),
                           pin_out(np.empty(B, dtype=np.int32)), pin_out(np.empty(B, dtype=np.int32)), n)
    conv_buf = out_host.converged
    e2e_steps = max(3, min(args.steps, 10))
    e2e_ms = []
    res = None
    for k in range(2 + e2e_steps):
        flush.fill_(k & 0xFF)
        torch.cuda.synchronize(dev)
        out_host.converged = conv_buf
        res = dec.decode(pin_noisy, pin_syn, args.e, out=out_host)
        if k >= 2:
            e2e_ms.append(dec.last_timing(e2e=True)[1])
    e2e_good = int((res.converged & np.all(res.corrected == fb.keys, axis=1)).sum()) * n
    e2e_total_ms = sum(e2e_ms)

    # ---- cross-rank aggregation: sums of work, max of time (shard.py) --------
    from paper_2001_07979_b200.shard import reduce_work_time

    (good_bits_all, e2e_good_all, frames_all), (total_ms_max, e2e_ms_max) = reduce_work_time(
        [float(good_bits), float(e2e_good * e2e_steps), float(B)], [total_ms, e2e_total_ms], device=dev)

    value = good_bits_all / (total_ms_max / 1e3) / 1e6
    e2e_value = e2e_good_all / (e2e_ms_max / 1e3) / 1e6

    # ---- roofline of the dominant kernel (the cooperative decode) ------------
    E = int(ens.matrices[0].edge_count) * u
    per_frame = [alg_bytes_per_frame(n, m, u, E, int(i)) for i in iters]
    alg_bytes = float(sum(per_frame))
    kms_mean = statistics.mean(kernel_ms)
    achieved = alg_bytes / (kms_mean / 1e3) / 1e9
    peak, peak_kind = measured_peak_hbm()
    traffic = None
    tf = ROOT / "profiles" / "decode_traffic.json"
    if tf.exists():
        try:
            t = json.loads(tf.read_text())
            if t.get("workload") == args.workload and t.get("frames") == B and t.get("e") == args.e:
                traffic = t.get("dram_bytes_per_launch")
        except Exception:
            pass

    # compute-side view: SFU (MUFU) operations of the check rule
    mufu_ops = float(sum(rule_evals(i) for i in iters)) * E * MUFU_PER_EDGE
    sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
    clocks_summary = clocks.summary()
    sm_mhz = clocks_summary.get("sm_mhz") or 1965.0
    mufu_peak = MUFU_PER_CLK_SM * sm_count * sm_mhz * 1e6
    mufu_ach = mufu_ops / (kms_mean / 1e3)

    line = {
        "metric": "reconciliation throughput (corrected Mbps)",
        "value": round(value, 3), "unit": "Mbps", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(total_ms_max / args.steps, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32" if args.precision == "fp32" else "f64",
        "data": "synthetic (reference Philox frame streams, "
                + ("synthetic random regular graphs)" if args.workload == "cfg4" else "PEG ensemble from the reference)"),
        "config": config_dict(args, ens),
        "fer": round(1.0 - float(conv.mean()), 6), "mean_iterations": round(float(iters.mean()), 4),
        "sweeps_run": sweeps,
        "e2e": {"value": round(e2e_value, 3), "unit": "Mbps",
                "h2d_bytes_per_step": int(fb.noisy.nbytes + pin_syn.nbytes + 8),
                "d2h_bytes_per_step": int(corrected.nbytes + 9 * B),
                "timing": "CUDA events on the workspace stream around mbp_decode_batch (host pinned buffers)"},
        "gpu_launches": 5 * args.steps,
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic,
                     "kernel": "mbp::decode_scatter_kernel (cooperative, persistent, all sweeps)",
                     "kernel_ms": round(kms_mean, 4), "alg_bytes_per_launch": alg_bytes,
                     "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                     "note": "achieved = SURVEY 8(d) message-streaming bytes / kernel time; the scatter "
                             "kernel keeps sweep-1/2 messages out of HBM, so frac > 1 is possible and "
                             "`traffic` (ncu DRAM bytes) is the real traffic",
                     "compute": {"unit": "MUFU op/s", "achieved": round(mufu_ach / 1e12, 4),
                                 "peak": round(mufu_peak / 1e12, 4), "scale": "1e12",
                                 "frac": round(mufu_ach / mufu_peak, 4),
                                 "basis": f"{MUFU_PER_EDGE} SFU ops per edge per Eq. 6 evaluation, "
                                          f"{MUFU_PER_CLK_SM}/clk/SM x {sm_count} SMs x median SM clock"}},
        "clocks": clocks_summary,
    }

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        corrected_c, conv_c, _, wall, frames_c, threads = cpu_decode_sample(ens, fb.noisy, pin_syn, args.e)
        good_c = conv_c & np.all(corrected_c == fb.keys[:frames_c], axis=1)
        line["cpu_baseline"] = {"value": round(int(good_c.sum()) * n / wall / 1e6, 4), "unit": "Mbps",
                                "cores": threads, "kind": "port",
                                "sample": f"first {frames_c} of the {B} frames, oracle/mbp_oracle.c "
                                          f"(reference decode_loop restated in C/libm fp64) on {threads} threads, "
                                          f"{wall:.1f} s wall"}
    if rank == 0 and not args.no_sweep:
        sweep = {}
        for e in (0.02, 0.04, 0.05):
            _, fbe = load_workload(rank, B, e, world, args.workload)
            syn_e = dec.syndromes(torch.from_numpy(fbe.keys).to(dev))
            nd = torch.from_numpy(fbe.noisy).to(dev)
            ed = torch.tensor([e], dtype=torch.float64, device=dev)
            dec.decode_device(nd, syn_e, ed, out=out)
            ts = []
            for k in range(5):
                flush.fill_(k)
                s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s0.record(stream)
                dec.decode_device(nd, syn_e, ed, out=out)
                s1.record(stream)
                torch.cuda.synchronize(dev)
                ts.append(s0.elapsed_time(s1))
            ok = out[1].cpu().numpy().astype(bool) & np.all(out[0].cpu().numpy() == fbe.keys, axis=1)
            sweep[str(e)] = {"mbps": round(int(ok.sum()) * n / (statistics.mean(ts) / 1e3) / 1e6, 1),
                             "fer": round(1 - float(out[1].cpu().numpy().mean()), 6),
                             "mean_iterations": round(float(out[2].cpu().numpy().mean()), 3)}
        line["qber_sweep"] = sweep
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
