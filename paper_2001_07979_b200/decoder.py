"""Multi-matrix belief-propagation (MBP) decoder on B200 -- the drop-in API.

Same module-level names and semantics as the reference decoder
(pkg/src/mmrecon/decoder.py:37-274, re-exported at __init__.py:14-21):
``DecoderConfig``, ``DecodeResult``, ``DecoderWorkspace``,
``compute_syndrome``, ``init_priors``, ``c2v_update``, ``v2c_update``,
``soft_decision``, ``decode``, ``reset`` -- with every decode executed by the
CUDA library (libmbp_b200.so, include/mbp.h).  Added: ``decode_batch`` /
``syndrome_batch`` and ``BatchDecoder`` for many frames per launch, the way
the hardware wants to be used.

Numerics: ``DecoderConfig.precision`` selects fp32 messages with Eq. 6 in the
phi domain (default, the production path) or fp64 messages with the
reference's literal tanh product ("fp64", parity mode).  Both follow the
reference's update order and stopping rule; see DESIGN.md §3 for the parity
contract each meets.
"""

from __future__ import annotations

import ctypes as C
import math
import threading
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .bits import BitBlock
from .matrix import stacked_layout

__all__ = [
    "DecoderConfig",
    "DecoderWorkspace",
    "DecodeResult",
    "BatchResult",
    "BatchDecoder",
    "DeviceEnsemble",
    "compute_syndrome",
    "init_priors",
    "c2v_update",
    "v2c_update",
    "soft_decision",
    "decode",
    "decode_batch",
    "syndrome_batch",
    "reset",
]

COMBINING_MODES = ("joint-graph", "isolated-per-matrix")
PRECISIONS = ("fp32", "fp64")


@dataclass(frozen=True)
class DecoderConfig:
    """decoder.py:53-68 plus ``precision`` (device arithmetic)."""

    max_iterations: int = 60
    llr_clamp: float = 30.0
    damping: float = 0.0
    combining_mode: str = "joint-graph"
    precision: str = "fp32"

    def __post_init__(self):
        if self.max_iterations < 1:
            raise ValueError(f"max_iterations must be >= 1, got {self.max_iterations}")
        if not self.llr_clamp > 0:
            raise ValueError(f"llr_clamp must be positive, got {self.llr_clamp}")
        if not 0.0 <= self.damping <= 1.0:
            raise ValueError(f"damping must be in [0, 1], got {self.damping}")
        if self.combining_mode not in COMBINING_MODES:
            raise ValueError(f"combining_mode must be one of {COMBINING_MODES}")
        if self.precision not in PRECISIONS:
            raise ValueError(f"precision must be one of {PRECISIONS}")

    def to_c(self, flags: int = 0) -> N.DecoderConfigC:
        return N.DecoderConfigC(
            int(self.max_iterations),
            N.MBP_JOINT_GRAPH if self.combining_mode == "joint-graph" else N.MBP_ISOLATED_PER_MATRIX,
            N.MBP_FP32_PHI if self.precision == "fp32" else N.MBP_FP64_TANH,
            int(flags), float(self.llr_clamp), float(self.damping))


def _cfg_of(config) -> DecoderConfig:
    """Accept ours, the reference's DecoderConfig, or None."""
    if config is None:
        return DecoderConfig()
    if isinstance(config, DecoderConfig):
        return config
    return DecoderConfig(config.max_iterations, config.llr_clamp, config.damping,
                         config.combining_mode, getattr(config, "precision", "fp32"))


@dataclass(frozen=True)
class DecodeResult:
    corrected: BitBlock
    converged: bool
    iterations_used: int
    residual_syndrome_mismatches: int
    decision_history: np.ndarray | None = None


@dataclass
class BatchResult:
    """Per-frame outputs of a batched decode (rows are BitBlock bytes)."""

    corrected: np.ndarray    # u8[B, ceil(n/8)]
    converged: np.ndarray    # bool[B]
    iterations: np.ndarray   # i32[B]
    mismatches: np.ndarray   # i32[B]
    n: int

    def result(self, k: int) -> DecodeResult:
        return DecodeResult(BitBlock(self.corrected[k].copy(), self.n), bool(self.converged[k]),
                            int(self.iterations[k]), int(self.mismatches[k]))


# ---------------------------------------------------------------------------
# device objects
# ---------------------------------------------------------------------------

class DeviceEnsemble:
    """H_1..H_u uploaded to one GPU as the stacked edge layout (mbp_ensemble)."""

    def __init__(self, ensemble, device: int = 0):
        self.layout = stacked_layout(ensemble)
        lay = self.layout
        self.n, self.m, self.u = lay.n, lay.m, lay.u
        self.device = int(device)
        self._ensemble = ensemble
        handle = C.c_void_p()
        chk_ptr = np.ascontiguousarray(lay.chk_ptr, dtype=np.int64)
        chk_var = np.ascontiguousarray(lay.chk_var, dtype=np.int32)
        N.call("mbp_ensemble_create", lay.n, lay.m, lay.u, chk_ptr.ctypes.data,
               chk_var.ctypes.data, self.device, C.byref(handle))
        self.handle = handle
        info = N.EnsembleInfoC()
        N.call("mbp_ensemble_get_info", self.handle, C.byref(info))
        self.info = info

    @property
    def nbytes_key(self) -> int:
        return (self.n + 7) // 8

    @property
    def nbytes_syn(self) -> int:
        return self.u * ((self.m + 7) // 8)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and N._LIB is not None:
            N._LIB.mbp_ensemble_destroy(h)
            self.handle = None


_DEV_CACHE_SIZE = 8
_DEV_CACHE: "OrderedDict" = OrderedDict()
_DEV_LOCK = threading.Lock()


def _content_key(ensemble) -> tuple:
    """Identity of a matrix set by content (memoised SHA-256 per matrix):
    equal graphs share one device upload whatever Python object holds them."""
    return tuple(h.content_hash() for h in _matrices(ensemble))


def device_ensemble(ensemble, device: int = 0) -> DeviceEnsemble:
    """Upload once per (matrix contents, device); the ensemble is immutable.
    The cache is a bounded LRU -- evicting only drops the cache's reference,
    a DeviceEnsemble lives as long as the BatchDecoders that use it."""
    if isinstance(ensemble, DeviceEnsemble):
        return ensemble
    key = (_content_key(ensemble), int(device))
    with _DEV_LOCK:
        de = _DEV_CACHE.get(key)
        if de is None:
            de = DeviceEnsemble(ensemble, device)
            _DEV_CACHE[key] = de
            while len(_DEV_CACHE) > _DEV_CACHE_SIZE:
                _DEV_CACHE.popitem(last=False)
        else:
            _DEV_CACHE.move_to_end(key)
        return de


class BatchDecoder:
    """A device workspace for up to ``max_frames`` frames (mbp_workspace).

    ``decode`` takes numpy rows (host path: copies in, decodes, copies out,
    synchronises) or CUDA tensors (device path: enqueued on the current torch
    stream, no synchronisation)."""

    def __init__(self, ensemble, max_frames: int, config=None, device: int = 0, flags: int = 0):
        self.dev = device_ensemble(ensemble, device)
        self.config = _cfg_of(config)
        self.flags = int(flags)
        self.max_frames = int(max_frames)
        handle = C.c_void_p()
        cfg = self.config.to_c(self.flags)
        N.call("mbp_workspace_create", self.dev.handle, self.max_frames, C.byref(cfg), C.byref(handle))
        self.handle = handle

    def configure(self, config=None, flags: int | None = None) -> None:
        config = _cfg_of(config)
        if flags is not None:
            self.flags = int(flags)
        cfg = config.to_c(self.flags)
        N.call("mbp_workspace_configure", self.handle, C.byref(cfg))
        self.config = config

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and N._LIB is not None:
            N._LIB.mbp_workspace_destroy(h)
            self.handle = None

    # -- host buffers -------------------------------------------------------
    def _check_rows(self, noisy, syn):
        B = noisy.shape[0]
        if noisy.shape != (B, self.dev.nbytes_key):
            raise ValueError(f"noisy rows must be [B, {self.dev.nbytes_key}] bytes, got {tuple(noisy.shape)}")
        if syn.shape != (B, self.dev.nbytes_syn):
            raise ValueError(f"syndrome rows must be [B, {self.dev.nbytes_syn}] bytes, got {tuple(syn.shape)}")
        return B

    def decode(self, noisy, syn, e, out=None, stream=None) -> BatchResult:
        if hasattr(noisy, "is_cuda") and noisy.is_cuda:
            return self.decode_device(noisy, syn, e, out=out, stream=stream)
        noisy = np.ascontiguousarray(noisy, dtype=np.uint8)
        syn = np.ascontiguousarray(syn, dtype=np.uint8)
        B = self._check_rows(noisy, syn)
        ev = np.ascontiguousarray(np.asarray(e, dtype=np.float64).reshape(-1))
        if ev.size not in (1, B):
            raise ValueError("e must be a scalar or one value per frame")
        if np.any(~((ev > 0.0) & (ev < 0.5))):
            raise ValueError(f"crossover probability must be in (0, 0.5), got {ev[(ev <= 0) | (ev >= 0.5)][0]}")
        if out is None:
            out = BatchResult(np.empty_like(noisy), np.empty(B, dtype=np.uint8),
                              np.empty(B, dtype=np.int32), np.empty(B, dtype=np.int32), self.dev.n)
        else:   # caller-owned (e.g. pinned) buffers are written in place
            for a, nm, dts, shp in ((out.corrected, "corrected", (np.uint8,), noisy.shape),
                                    (out.converged, "converged", (np.uint8, np.bool_), (B,)),
                                    (out.iterations, "iterations", (np.int32,), (B,)),
                                    (out.mismatches, "mismatches", (np.int32,), (B,))):
                if (not isinstance(a, np.ndarray) or a.dtype.type not in dts or a.shape[:len(shp)] != tuple(shp)
                        or a.shape[0] != shp[0] or not a.flags.c_contiguous or not a.flags.writeable):
                    raise ValueError(f"out.{nm} must be a writeable contiguous {dts[0].__name__} array of "
                                     f"shape {tuple(shp)}")
        N.call("mbp_decode_batch", self.handle, noisy.ctypes.data, syn.ctypes.data, ev.ctypes.data,
               0 if ev.size == 1 else 1, B, N.ptr(out.corrected), N.ptr(out.converged),
               N.ptr(out.iterations), N.ptr(out.mismatches))
        # a bool VIEW of the same (possibly pinned) bytes: the buffer stays the
        # caller's, so a reused `out` keeps copying into pinned memory
        out.converged = out.converged.view(np.bool_)
        return out

    def _check_device_tensor(self, t, name, dtype, shape=None):
        import torch

        if not torch.is_tensor(t) or not t.is_cuda:
            raise ValueError(f"{name} must be a CUDA tensor")
        if t.device.index != self.dev.device:
            raise ValueError(f"{name} is on cuda:{t.device.index}, the ensemble on cuda:{self.dev.device}")
        if t.dtype != dtype:
            raise ValueError(f"{name} must have dtype {dtype}, got {t.dtype}")
        if not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
        if shape is not None and tuple(t.shape) != tuple(shape):
            raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")

    def decode_device(self, noisy, syn, e, out=None, stream=None):
        """CUDA-tensor path (inputs resident in HBM); returns device tensors.

        ``noisy``/``syn``: contiguous uint8 rows on the ensemble's device; ``e``
        a float in (0, 0.5) or a contiguous float64 CUDA tensor of 1 or B
        values (not range-checked: that would need a device sync)."""
        import torch

        self._check_device_tensor(noisy, "noisy", torch.uint8)
        B = self._check_rows(noisy, syn)
        self._check_device_tensor(syn, "syn", torch.uint8)
        if not torch.is_tensor(e):
            e = float(e)
            if not 0.0 < e < 0.5:
                raise ValueError(f"crossover probability must be in (0, 0.5), got {e}")
            e = torch.tensor([e], dtype=torch.float64, device=noisy.device)
        self._check_device_tensor(e, "e", torch.float64)
        if e.numel() not in (1, B):
            raise ValueError("e must be a scalar or one value per frame")
        if out is None:
            out = (torch.empty_like(noisy), torch.empty(B, dtype=torch.uint8, device=noisy.device),
                   torch.empty(B, dtype=torch.int32, device=noisy.device),
                   torch.empty(B, dtype=torch.int32, device=noisy.device))
        else:
            for t, nm, dt, shp in zip(out, ("corrected", "converged", "iterations", "mismatches"),
                                      (torch.uint8, torch.uint8, torch.int32, torch.int32),
                                      (tuple(noisy.shape), (B,), (B,), (B,))):
                self._check_device_tensor(t, f"out.{nm}", dt, shp)
        s = stream if stream is not None else torch.cuda.current_stream(noisy.device).cuda_stream
        N.call("mbp_decode_batch_device", self.handle, noisy.data_ptr(), syn.data_ptr(), e.data_ptr(),
               0 if e.numel() == 1 else 1, B, out[0].data_ptr(), out[1].data_ptr(), out[2].data_ptr(),
               out[3].data_ptr(), C.c_void_p(s))
        return out

    def syndromes(self, keys, out=None, stream=None):
        """Alice side, Eq. 1 for all u matrices: rows [B, u*ceil(m/8)]."""
        if hasattr(keys, "is_cuda") and keys.is_cuda:
            import torch

            self._check_device_tensor(keys, "keys", torch.uint8)
            B = keys.shape[0]
            if keys.shape != (B, self.dev.nbytes_key):
                raise ValueError(f"key rows must be [B, {self.dev.nbytes_key}] bytes")
            if out is None:
                out = torch.empty((B, self.dev.nbytes_syn), dtype=torch.uint8, device=keys.device)
            self._check_device_tensor(out, "out", torch.uint8, (B, self.dev.nbytes_syn))
            s = stream if stream is not None else torch.cuda.current_stream(keys.device).cuda_stream
            N.call("mbp_syndrome_batch_device", self.handle, keys.data_ptr(), B, out.data_ptr(), C.c_void_p(s))
            return out
        keys = np.ascontiguousarray(keys, dtype=np.uint8)
        B = keys.shape[0]
        if keys.shape != (B, self.dev.nbytes_key):
            raise ValueError(f"key rows must be [B, {self.dev.nbytes_key}] bytes")
        out = np.empty((B, self.dev.nbytes_syn), dtype=np.uint8) if out is None else out
        N.call("mbp_syndrome_batch", self.handle, keys.ctypes.data, B, out.ctypes.data)
        return out

    # -- state of the last decode ----------------------------------------------
    def posterior(self, k: int) -> np.ndarray:
        out = np.empty(self.dev.n, dtype=np.float64)
        N.call("mbp_workspace_read_posterior", self.handle, int(k), out.ctypes.data)
        return out

    def c2v(self, k: int) -> np.ndarray:
        out = np.empty(self.dev.layout.edges, dtype=np.float64)
        N.call("mbp_workspace_read_c2v", self.handle, int(k), out.ctypes.data)
        return out

    def v2c_previous(self, k: int) -> np.ndarray:
        out = np.empty(self.dev.layout.edges, dtype=np.float64)
        N.call("mbp_workspace_read_v2c", self.handle, int(k), out.ctypes.data)
        return out

    def history(self, k: int, rows: int) -> np.ndarray:
        nb = self.dev.nbytes_key
        out = np.zeros((rows, nb), dtype=np.uint8)
        N.call("mbp_workspace_read_history", self.handle, int(k), int(rows), out.ctypes.data)
        return np.unpackbits(out, axis=1, count=self.dev.n, bitorder="little")

    def phase_times(self) -> dict:
        """Per-phase device time (ms) of the last decode chunk
        (needs flags MBP_PROFILE_PHASES): check / variable / syndrome phase
        totals over the executed sweeps, the initial check and the tail."""
        cap = 3 * (self.config.max_iterations + 1) + 8
        buf = np.zeros(cap, dtype=np.uint64)
        cnt = C.c_int32(0)
        N.call("mbp_workspace_read_phase_times", self.handle, buf.ctypes.data, cap, C.byref(cnt))
        k = min(cnt.value, cap - 4)
        ts = buf[:k].astype(np.float64) / 1e6
        cts = buf[k:k + 4].astype(np.float64) / 1e6
        d = np.diff(ts)
        sweeps = (len(ts) - 3) // 3
        out = {"sweeps": sweeps, "total_ms": float(ts[-1] - ts[0]), "syncheck0_ms": float(d[0])}
        if sweeps:
            body = d[1:1 + 3 * sweeps].reshape(sweeps, 3)
            out.update(check_ms=body[:, 0].tolist(), var_ms=body[:, 1].tolist(), syncheck_ms=body[:, 2].tolist())
        out["tail_ms"] = float(d[-1]) if len(d) > 1 else 0.0
        if cts[0] > 0:
            cd = np.diff(cts)
            out["compaction_ms"] = {"maps": float(cd[0]), "move": float(cd[1]), "barrier": float(cd[2])}
            # the compaction runs between a sweep's first stamp and its check
            # phase: report that check phase without it
            for i in range(sweeps):
                if ts[1 + 3 * i] <= cts[0] <= ts[2 + 3 * i]:
                    out["check_ms"][i] -= float(cts[3] - cts[0])
        return out

    def last_stats(self):
        """(sweeps run, sweep at which frames were compacted or 0) of the last chunk."""
        sw = C.c_int32(0)
        cs = C.c_int32(0)
        N.call("mbp_workspace_last_stats", self.handle, C.byref(sw), C.byref(cs))
        return int(sw.value), int(cs.value)

    def last_timing(self, e2e: bool = False):
        """(decode-kernel ms, sweeps run) of the last decode; with e2e=True
        also the device-timed ms of the last host-buffer call."""
        ms = C.c_float(0.0)
        e2 = C.c_float(0.0)
        sw = C.c_int32(0)
        N.call("mbp_workspace_last_timing", self.handle, C.byref(ms), C.byref(e2) if e2e else None,
               C.byref(sw))
        if e2e:
            return float(ms.value), float(e2.value), int(sw.value)
        return float(ms.value), int(sw.value)


def decode_batch(ensemble, noisy_rows, syn_rows, e, config=None, device: int = 0) -> BatchResult:
    """Decode B frames in one launch (host rows in, host rows out)."""
    noisy_rows = np.ascontiguousarray(noisy_rows, dtype=np.uint8)
    dec = BatchDecoder(ensemble, max(noisy_rows.shape[0], 1), config, device)
    return dec.decode(noisy_rows, syn_rows, e)


def syndrome_batch(ensemble, key_rows, device: int = 0) -> np.ndarray:
    key_rows = np.ascontiguousarray(key_rows, dtype=np.uint8)
    dec = BatchDecoder(ensemble, max(key_rows.shape[0], 1), None, device)
    return dec.syndromes(key_rows)


# ---------------------------------------------------------------------------
# reference API mirror
# ---------------------------------------------------------------------------

class DecoderWorkspace:
    """Per-frame message buffers for one ensemble (decoder.py:80-134).

    Host float64 arrays with the reference's stacked layout; after ``decode``
    they hold the final state as the reference's would (posterior, c2v, v2c,
    hard).  ``decode`` runs the production (scatter) kernel, which keeps no
    messages; the message arrays are materialised on first access by
    replaying the frame on the explicit-message kernel (same decisions, same
    iteration count -- tests/test_gpu_scatter.py), so callers that never read
    them (bench.measure_throughput, session._decode_block) do not pay for
    it."""

    def __init__(self, ensemble, config=None):
        self.ensemble = ensemble
        self.config = _cfg_of(config)
        lay = stacked_layout(ensemble)
        self.layout = lay
        self.edge_off = lay.edge_off
        self.chk_ptr = lay.chk_ptr
        self.chk_var = lay.chk_var
        self.var_ptr = lay.var_ptr
        self.var_edge = lay.var_edge
        total = lay.edges
        n = lay.n
        self._v2c = np.zeros(total, dtype=np.float64)
        self._c2v = np.zeros(total, dtype=np.float64)
        self.priors = np.zeros(n, dtype=np.float64)
        self._posterior = np.zeros(n, dtype=np.float64)
        self.hard = np.zeros(n, dtype=np.uint8)
        self.iteration = 0
        self._dec = None
        self._dec_key = None
        self._fast = None
        self._fast_key = None
        self._pending = None     # (noisy row, syndrome row, e, config) of a decode not yet mirrored

    # message state, materialised on demand
    def _state(self, name):
        if self._pending is not None:
            _materialize(self)
        return getattr(self, name)

    def _set_state(self, name, value):
        if self._pending is not None:
            _materialize(self)
        getattr(self, name)[...] = value

    v2c = property(lambda self: self._state("_v2c"), lambda self, v: self._set_state("_v2c", v))
    c2v = property(lambda self: self._state("_c2v"), lambda self, v: self._set_state("_c2v", v))
    posterior = property(lambda self: self._state("_posterior"), lambda self, v: self._set_state("_posterior", v))

    def reset(self) -> None:
        self._pending = None
        self._v2c[:] = 0.0
        self._c2v[:] = 0.0
        self.priors[:] = 0.0
        self._posterior[:] = 0.0
        self.hard[:] = 0
        self.iteration = 0

    def matrix_slice(self, l: int) -> slice:
        return slice(int(self.edge_off[l]), int(self.edge_off[l + 1]))

    def _device(self, config: DecoderConfig, track: bool) -> BatchDecoder:
        # state readback: the explicit-message kernel with kept state
        flags = N.MBP_KEEP_STATE | N.MBP_EXPLICIT_MESSAGES | (N.MBP_RECORD_HISTORY if track else 0)
        shape_key = (config.precision, config.combining_mode)
        if self._dec is None or self._dec_key != shape_key:
            self._dec = BatchDecoder(self.ensemble, 1, config, flags=flags)
            self._dec_key = shape_key
        elif self._dec.config != config or self._dec.flags != flags:
            self._dec.configure(config, flags)
        return self._dec

    def _production(self, config: DecoderConfig, track: bool) -> BatchDecoder:
        # decisions only: the production path, no kept state
        flags = N.MBP_RECORD_HISTORY if track else 0
        shape_key = (config.precision, config.combining_mode)
        if self._fast is None or self._fast_key != shape_key:
            self._fast = BatchDecoder(self.ensemble, 1, config, flags=flags)
            self._fast_key = shape_key
        elif self._fast.config != config or self._fast.flags != flags:
            self._fast.configure(config, flags)
        return self._fast


def _materialize(ws: DecoderWorkspace) -> None:
    """Mirror the final device state of the last decode into the workspace
    arrays: replay the frame on the explicit-message kernel with kept state."""
    noisy, syn, e, config, iters = ws._pending
    ws._pending = None
    lay = ws.layout
    if iters == 0:
        ws._v2c[:] = ws.priors[lay.chk_var]
        ws._c2v[:] = 0.0
        ws._posterior[:] = 0.0
        return
    dec = ws._device(config, False)
    dec.decode(noisy, syn, e)
    ws._c2v[:] = dec.c2v(0)
    ws._posterior[:] = dec.posterior(0)
    ws._v2c[:] = _final_v2c(ws, config, dec)


def _matrices(ensemble_or_matrix):
    return tuple(getattr(ensemble_or_matrix, "matrices", (ensemble_or_matrix,)))


def compute_syndrome(matrix, key) -> BitBlock:
    """z_j = XOR of key bits over check j (Eq. 1) -- on the GPU.  Thread-safe:
    the reference calls it from worker threads (bench._frame_inputs), so each
    cached syndrome workspace is used under its own lock."""
    if key.length != matrix.n:
        raise ValueError(f"key length {key.length} != n={matrix.n}")
    dec, lock = _syndrome_decoder(matrix)
    with lock:
        rows = dec.syndromes(np.asarray(key.data, dtype=np.uint8).reshape(1, -1))
    return BitBlock(rows[0, : (matrix.m + 7) // 8].copy(), matrix.m)


_SYN_CACHE: "OrderedDict" = OrderedDict()
_SYN_LOCK = threading.Lock()


def _syndrome_decoder(matrix):
    """(BatchDecoder, lock) per matrix contents; bounded LRU like _DEV_CACHE."""
    key = _content_key(matrix)
    with _SYN_LOCK:
        ent = _SYN_CACHE.get(key)
        if ent is None:
            ent = (BatchDecoder(matrix, 32), threading.Lock())
            _SYN_CACHE[key] = ent
            while len(_SYN_CACHE) > _DEV_CACHE_SIZE:
                _SYN_CACHE.popitem(last=False)
        else:
            _SYN_CACHE.move_to_end(key)
        return ent


def init_priors(noisy_key, e: float) -> np.ndarray:
    """(1 - 2 y_i) ln((1-e)/e) (Eq. 5; decoder.py:147-152).  Host helper: the
    device decode forms the same prior itself from the packed noisy key."""
    if not 0.0 < e < 0.5:
        raise ValueError(f"crossover probability must be in (0, 0.5), got {e}")
    bits = noisy_key.to_bits().astype(np.float64)
    return (1.0 - 2.0 * bits) * math.log((1.0 - e) / e)


def _precision_code(ws) -> int:
    return N.MBP_FP64_TANH if ws.config.precision == "fp64" else N.MBP_FP32_PHI


def c2v_update(workspace: DecoderWorkspace, matrix_index: int, syndrome) -> None:
    """Recompute matrix ``matrix_index``'s c2v messages from ws.v2c (Eq. 6)."""
    m = workspace.layout.m
    if syndrome.length != m:
        raise ValueError(f"syndrome length {syndrome.length} != m={m}")
    dev = device_ensemble(workspace.ensemble)
    syn = np.ascontiguousarray(syndrome.to_bits(), dtype=np.uint8)
    N.call("mbp_c2v_pass", dev.handle, _precision_code(workspace), int(matrix_index), syn.ctypes.data,
           float(workspace.config.llr_clamp), workspace.v2c.ctypes.data, workspace.c2v.ctypes.data)


def v2c_update(workspace: DecoderWorkspace, matrix_index: int) -> None:
    cfg = workspace.config
    dev = device_ensemble(workspace.ensemble)
    N.call("mbp_v2c_pass", dev.handle, _precision_code(workspace), int(matrix_index),
           int(cfg.combining_mode == "joint-graph"), float(cfg.damping), float(cfg.llr_clamp),
           workspace.c2v.ctypes.data, workspace.priors.ctypes.data, workspace.v2c.ctypes.data)


def soft_decision(workspace: DecoderWorkspace) -> np.ndarray:
    """Posterior LLR (Eq. 2): prior + every matrix's c2v."""
    dev = device_ensemble(workspace.ensemble)
    N.call("mbp_posterior_pass", dev.handle, _precision_code(workspace), workspace.c2v.ctypes.data,
           workspace.priors.ctypes.data, workspace.posterior.ctypes.data)
    return workspace.posterior


def reset(workspace: DecoderWorkspace) -> None:
    workspace.reset()


def _same_ensemble(a, b) -> bool:
    if a is b:
        return True
    ma, mb = _matrices(a), _matrices(b)
    return len(ma) == len(mb) and all(x == y for x, y in zip(ma, mb))


def decode(ensemble, noisy_key, syndromes, e: float, config=None, workspace=None,
           track_decisions: bool = False) -> DecodeResult:
    """Correct ``noisy_key`` toward the key behind ``syndromes`` (decoder.py:207-274).

    A batch-of-one call of the device decoder; the workspace's host arrays
    mirror the final device state as the reference's would."""
    config = _cfg_of(config)
    mats = _matrices(ensemble)
    n, m, u = mats[0].n, mats[0].m, len(mats)
    if noisy_key.length != n:
        raise ValueError(f"key length {noisy_key.length} != n={n}")
    if len(syndromes) != u:
        raise ValueError(f"{len(syndromes)} syndromes for u={u} matrices")
    for l, z in enumerate(syndromes):
        if z.length != m:
            raise ValueError(f"syndrome {l} length {z.length} != m={m}")
    if not 0.0 < e < 0.5:
        raise ValueError(f"crossover probability must be in (0, 0.5), got {e}")
    noisy = np.asarray(noisy_key.data, dtype=np.uint8).reshape(1, -1)
    syn = np.concatenate([np.asarray(z.data, dtype=np.uint8) for z in syndromes]).reshape(1, -1)
    if workspace is None:
        # nothing to mirror: a per-thread production decoder, no state kept
        dec = _thread_decoder(ensemble, config, track_decisions)
        res = dec.decode(noisy, syn, e)
        iters = int(res.iterations[0])
        return DecodeResult(
            corrected=BitBlock(res.corrected[0].copy(), n),
            converged=bool(res.converged[0]),
            iterations_used=iters,
            residual_syndrome_mismatches=int(res.mismatches[0]),
            decision_history=dec.history(0, iters + 1) if track_decisions else None,
        )
    if not _same_ensemble(workspace.ensemble, ensemble):
        raise ValueError("workspace was built for a different ensemble")
    workspace.config = config
    workspace.reset()
    workspace.priors[:] = init_priors(noisy_key, e)

    dec = workspace._production(config, track_decisions)
    res = dec.decode(noisy, syn, e)
    iters = int(res.iterations[0])
    workspace.hard[:] = np.unpackbits(res.corrected[0], count=n, bitorder="little")
    workspace.iteration = iters
    # the message arrays follow on first access (DecoderWorkspace._state)
    workspace._pending = (noisy.copy(), syn.copy(), float(e), config, iters)
    history = dec.history(0, iters + 1) if track_decisions else None
    return DecodeResult(
        corrected=BitBlock(res.corrected[0].copy(), n),
        converged=bool(res.converged[0]),
        iterations_used=iters,
        residual_syndrome_mismatches=int(res.mismatches[0]),
        decision_history=history,
    )


_TLS = threading.local()


def _thread_decoder(ensemble, config: DecoderConfig, track: bool) -> BatchDecoder:
    """A one-frame production decoder per (thread, matrix set, precision,
    combining mode): decode() without a workspace is called from worker
    threads (the reference's measure_throughput, session._decode_block), and
    a device workspace must not be shared between threads."""
    cache = getattr(_TLS, "decoders", None)
    if cache is None:
        cache = _TLS.decoders = OrderedDict()
    key = (_content_key(ensemble), config.precision, config.combining_mode)
    dec = cache.get(key)
    flags = N.MBP_RECORD_HISTORY if track else 0
    if dec is None:
        dec = BatchDecoder(ensemble, 1, config, flags=flags)
        cache[key] = dec
        while len(cache) > 4:
            cache.popitem(last=False)
    elif dec.config != config or dec.flags != flags:
        dec.configure(config, flags)
    return dec


def _final_v2c(ws: DecoderWorkspace, cfg: DecoderConfig, dec: BatchDecoder) -> np.ndarray:
    """v2c after the last sweep's v2c_pass (_kernels.py:264-290), from the
    device's final c2v/posterior (and previous v2c when damping)."""
    lay = ws.layout
    if cfg.combining_mode == "joint-graph":
        total_e = ws.posterior[lay.chk_var]
    else:
        total_e = np.empty(lay.edges)
        for l in range(lay.u):
            sl = ws.matrix_slice(l)
            tot = ws.priors.copy()
            np.add.at(tot, lay.chk_var[sl], ws.c2v[sl])
            total_e[sl] = tot[lay.chk_var[sl]]
    val = total_e - ws.c2v
    if cfg.damping != 0.0:
        val = (1.0 - cfg.damping) * val + cfg.damping * dec.v2c_previous(0)
    return np.clip(val, -cfg.llr_clamp, cfg.llr_clamp)
