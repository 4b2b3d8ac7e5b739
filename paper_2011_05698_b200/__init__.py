"""B200-native sFFT4.0 hot path -- Python mirror of the reference interface.

The reference entry point (proj/include/msfft/sfft4.hpp:64-65)

    SfftResult sfft4(const ComplexSignal& x, int64_t k,
                     const MultiscaleConfig& cfg, uint64_t seed,
                     double delta = 1e-8);

is mirrored by :func:`sfft4` with the same argument meaning and the same
error behaviour: ``std::invalid_argument`` -> :class:`InvalidArgument`
(a ``ValueError``) and ``std::domain_error`` -> :class:`DomainError`, with the
reference's messages.  Everything runs through ``libmsfft_b200.so`` (the
C ABI in ``include/msfft_b200.h``); there is no CPU fallback.

:class:`Plan` is the batched form (independent signals sharing n, k, l, q,
delta; one seed each), used for the batched-throughput configuration.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib as _L

__all__ = [
    "MultiscaleConfig", "TransformStats", "SparseSpectrum", "SfftResult", "sfft4", "Plan",
    "window", "window_response", "trace", "InvalidArgument", "DomainError", "CudaError",
    "splitmix64", "device_count",
]


class InvalidArgument(ValueError):
    """std::invalid_argument in the reference."""


class DomainError(ArithmeticError):
    """std::domain_error escaping the reference's sfft4."""


class CudaError(RuntimeError):
    """No usable CUDA device, or a CUDA failure (there is no CPU fallback)."""


def _raise(status: int, err) -> None:
    if status == _L.MSFFT_OK:
        return
    msg = err.value.decode(errors="replace") if err is not None else ""
    if status == _L.MSFFT_ERR_INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    if status == _L.MSFFT_ERR_DOMAIN:
        raise DomainError(msg)
    if status == _L.MSFFT_ERR_CUDA:
        raise CudaError(msg)
    raise RuntimeError(msg)


def splitmix64(x: int) -> int:
    """splitmix64 (proj/include/msfft/rng.hpp:9-14): seed derivation used by
    the reference bench (algo seed = splitmix64(seed ^ 0x53), bench.cpp:117)."""
    m = (1 << 64) - 1
    x = (x + 0x9E3779B97F4A7C15) & m
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & m
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & m
    return x ^ (x >> 31)


@dataclass
class MultiscaleConfig:
    """proj/include/msfft/locate.hpp:13-19."""
    l: int = 16
    q: float = 1.0

    def shrink(self) -> float:
        return float(self.l) / (self.q + 1.0)

    def validate(self) -> None:
        if self.l < 2:
            raise InvalidArgument("MultiscaleConfig: l must be >= 2")
        if self.q < 0.0:
            raise InvalidArgument("MultiscaleConfig: q must be >= 0")
        if not (self.shrink() > 1.0):
            raise InvalidArgument("MultiscaleConfig: l/(q+1) must exceed 1")


@dataclass
class TransformStats:
    """proj/include/msfft/sfft4.hpp:32-40 (runtime_ms is device time)."""
    samples_used: int = 0
    samples_round_sum: int = 0
    sample_fraction: float = 0.0
    runtime_ms: float = 0.0
    iterations: int = 0
    b_first: int = 0
    stage_counts: list = field(default_factory=list)

    @classmethod
    def _from(cls, s: _L.Stats) -> "TransformStats":
        it = int(s.iterations)
        return cls(int(s.samples_used), int(s.samples_round_sum), float(s.sample_fraction),
                   float(s.runtime_ms), it, int(s.b_first), [int(v) for v in s.stage_counts[:it]])


@dataclass
class SparseSpectrum:
    """proj/include/msfft/signal.hpp:23-28; entries in ascending position."""
    n: int
    positions: np.ndarray
    coeffs: np.ndarray

    @property
    def entries(self) -> dict:
        return {int(f): complex(c) for f, c in zip(self.positions, self.coeffs)}


@dataclass
class SfftResult:
    spectrum: SparseSpectrum
    stats: TransformStats


def _torch_stream(device) -> int:
    """The current torch stream of `device` (its handle), so the split-phase
    calls order after the caller's producers."""
    import torch
    return int(torch.cuda.current_stream(device).cuda_stream)


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _signal_arg(x):
    """-> (pointer, n, dtype code, location, keepalive)."""
    if _is_torch(x):
        import torch
        if x.dtype not in (torch.complex64, torch.complex128):
            raise InvalidArgument("sfft4: x must be complex64 or complex128")
        if not x.is_contiguous():
            x = x.contiguous()
        dt = _L.MSFFT_C128 if x.dtype == torch.complex128 else _L.MSFFT_C64
        loc = _L.MSFFT_DEVICE if x.is_cuda else _L.MSFFT_HOST
        return C.c_void_p(x.data_ptr()), int(x.shape[-1]), dt, loc, x
    a = np.asarray(x)
    if a.dtype == np.complex64:
        dt = _L.MSFFT_C64
    else:
        a = a.astype(np.complex128, copy=False)
        dt = _L.MSFFT_C128
    a = np.ascontiguousarray(a)
    return C.c_void_p(a.ctypes.data), int(a.shape[-1]), dt, _L.MSFFT_HOST, a


def validate_signal(x, n: int | None = None, stream=None) -> float:
    """ComplexSignal::validate (proj/src/signal.cpp:18-26) for one signal or
    a (batch, n) array/tensor: n a power of two >= 4, sample count == n, all
    samples finite, else InvalidArgument with the reference's message.  CUDA
    tensors are scanned on the device (`stream`, default the legacy stream);
    returns the scan kernel's device ms (0 for host input)."""
    ptr, cnt, dt, loc, keep = _signal_arg(x)
    shape = tuple(keep.shape)
    batch = 1 if len(shape) == 1 else int(shape[0])
    nn = cnt if n is None else int(n)
    ms = C.c_double()
    err = C.create_string_buffer(1024)
    _raise(_L.lib().msfft_validate_signal(ptr, nn, cnt, batch, cnt, dt, loc,
                                          C.c_void_p(stream or 0), C.byref(ms), err, 1024), err)
    return ms.value


def device_count() -> int:
    return int(_L.lib().msfft_device_count())


def sfft4(x, k: int, cfg: MultiscaleConfig | None = None, seed: int = 0,
          delta: float = 1e-8) -> SfftResult:
    """Drop-in for msfft::sfft4 (proj/src/sfft4.cpp:131-187) on the GPU.

    x: 1-D complex array (numpy, or torch CPU/CUDA tensor), complex128 or
    complex64 (upcast exactly).  Returns the K-pruned spectrum in ascending
    position and the transform stats.
    """
    cfg = cfg or MultiscaleConfig()
    L = _L.lib()
    ptr, n, dt, loc, keep = _signal_arg(x)
    cap = max(int(k), 1)
    f = np.zeros(cap, np.int64)
    c = np.zeros(2 * cap, np.float64)
    cnt = C.c_int64()
    st = _L.Stats()
    err = C.create_string_buffer(1024)
    status = L.msfft_sfft4(ptr, n, dt, loc, int(k), int(cfg.l), float(cfg.q),
                           int(seed) & ((1 << 64) - 1), float(delta), cap,
                           f.ctypes.data_as(C.POINTER(C.c_int64)),
                           c.ctypes.data_as(C.POINTER(C.c_double)), C.byref(cnt), C.byref(st),
                           err, 1024)
    del keep
    _raise(status, err)
    m = cnt.value
    spec = SparseSpectrum(n, f[:m].copy(), c.view(np.complex128)[:m].copy())
    return SfftResult(spec, TransformStats._from(st))


class Plan:
    """Batched sfft4 over independent signals sharing (n, k, l, q, delta).

    Window design for the whole halving schedule happens here (cold path),
    as the reference pre-resolves windows before its timer
    (proj/src/sfft4.cpp:146-154).
    """

    def __init__(self, n: int, k: int, cfg: MultiscaleConfig | None = None,
                 delta: float = 1e-8, dtype: str = "complex64", device: int = -1):
        cfg = cfg or MultiscaleConfig()
        self.n, self.k, self.cfg, self.delta = int(n), int(k), cfg, float(delta)
        self.dtype = dtype
        dt = _L.MSFFT_C64 if dtype in ("complex64", "c64") else _L.MSFFT_C128
        self._lib = _L.lib()
        h = C.c_void_p()
        err = C.create_string_buffer(1024)
        _raise(self._lib.msfft_plan_create(self.n, self.k, int(cfg.l), float(cfg.q),
                                           self.delta, dt, int(device), C.byref(h), err, 1024),
               err)
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.msfft_plan_destroy(h)
            self._h = None

    def stats(self) -> TransformStats:
        s = _L.Stats()
        self._lib.msfft_plan_stats(self._h, C.byref(s))
        return TransformStats._from(s)

    def launches(self, batch: int, assume_valid: bool = False, serial: bool = False) -> int:
        flags = _L.MSFFT_FLAG_ASSUME_VALID if assume_valid else 0
        if serial:
            flags |= _L.MSFFT_FLAG_SERIAL
        return int(self._lib.msfft_plan_launches(self._h, int(batch), flags))

    def gather_traffic(self, seeds):
        """(samples loaded, distinct 32-B sectors) of the fused gather for
        these signals -- the algorithmic bytes behind the roofline."""
        seeds = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64).reshape(-1))
        a, b = C.c_int64(), C.c_int64()
        self._lib.msfft_plan_gather_traffic(self._h, seeds.size,
                                            seeds.ctypes.data_as(C.POINTER(C.c_uint64)),
                                            C.byref(a), C.byref(b))
        return a.value, b.value

    def stage_times(self):
        """[encode, bucket FFT (b > 256), decode] ms of the last execute run
        with stage_times=True."""
        ms = (C.c_double * 3)()
        self._lib.msfft_plan_stage_times(self._h, ms)
        return [float(v) for v in ms]

    def execute(self, x, seeds, out=None, assume_valid: bool = False, stream=None,
                stage_times: bool = False, serial: bool = False, async_: bool = False):
        """x: (batch, n) complex array/tensor (host or CUDA).  seeds: batch
        integers.  out: optional (f, c, count) preallocated outputs -- torch
        CUDA tensors (int64 [B,k], complex128 [B,k], int64 [B]) keep the
        results on the device; otherwise numpy arrays are returned.
        async_=True (CUDA x and out only) returns once the work is enqueued:
        outputs are ready when the stream reaches them and errors surface in
        sync().  Returns (f, c, count, device_ms) (device_ms 0 when async)."""
        ptr, n, dt, loc, keep = _signal_arg(x)
        if n != self.n:
            raise InvalidArgument("ComplexSignal: sample count != n")
        shape = tuple(keep.shape)
        batch = 1 if len(shape) == 1 else int(shape[0])
        seeds = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64).reshape(-1))
        if seeds.size != batch:
            raise InvalidArgument("Plan.execute: need one seed per signal")
        if out is None:
            f = np.zeros((batch, self.k), np.int64)
            c = np.zeros((batch, self.k), np.complex128)
            cnt = np.zeros(batch, np.int64)
            fptr, cptr, nptr = f.ctypes.data, c.ctypes.data, cnt.ctypes.data
            oloc = _L.MSFFT_HOST
        else:
            f, c, cnt = out
            if _is_torch(f):
                fptr, cptr, nptr = f.data_ptr(), c.data_ptr(), cnt.data_ptr()
                oloc = _L.MSFFT_DEVICE if f.is_cuda else _L.MSFFT_HOST
            else:
                fptr, cptr, nptr = f.ctypes.data, c.ctypes.data, cnt.ctypes.data
                oloc = _L.MSFFT_HOST
        ms = C.c_double()
        err = C.create_string_buffer(1024)
        flags = _L.MSFFT_FLAG_ASSUME_VALID if assume_valid else 0
        if serial:
            flags |= _L.MSFFT_FLAG_SERIAL
        if stage_times:
            flags |= _L.MSFFT_FLAG_STAGE_TIMES
        if async_:
            flags |= _L.MSFFT_FLAG_ASYNC
        status = self._lib.msfft_execute(
            self._h, batch, ptr, n, loc, seeds.ctypes.data_as(C.POINTER(C.c_uint64)),
            C.c_void_p(fptr), C.c_void_p(cptr), C.c_void_p(nptr), oloc, flags,
            C.c_void_p(stream or 0), C.byref(ms), err, 1024)
        _raise(status, err)
        return f, c, cnt, ms.value

    @property
    def ingest_samples_per_signal(self) -> int:
        """Samples per signal moved host->device for host inputs (sparse
        ingest); 0 when whole signals are copied."""
        return int(self._lib.msfft_plan_ingest_samples(self._h))

    def copy_bytes(self):
        """(host->device, device->host) bytes moved by the last execute."""
        a, b = C.c_int64(), C.c_int64()
        self._lib.msfft_plan_copy_bytes(self._h, C.byref(a), C.byref(b))
        return a.value, b.value

    def sync(self, stream=None) -> None:
        """Wait for this plan's work on `stream` and raise the errors of
        asynchronous execute calls since the last sync."""
        err = C.create_string_buffer(1024)
        _raise(self._lib.msfft_plan_sync(self._h, C.c_void_p(stream or 0), err, 1024), err)

    # ---- split phases: one signal sharded by index range over GPUs ----------
    @property
    def values_per_signal(self) -> int:
        """Bucket values per signal: sum over iterations of rounds x b."""
        return int(self._lib.msfft_plan_values_per_signal(self._h))

    def encode_values(self, x_local, seeds, x_lo: int, y=None, assume_valid: bool = False):
        """Partial bucket values of the samples x[x_lo, x_lo + span) held in
        x_local (CUDA tensor, (batch, span) or (span,)); the rest of the signal
        counts as 0.  Summing the results of ranks whose ranges tile [0, n)
        gives the full bucket vector (see paper_2011_05698_b200.dist).
        Returns y: complex128 CUDA tensor (batch, values_per_signal)."""
        import torch
        if not (_is_torch(x_local) and x_local.is_cuda):
            raise InvalidArgument("Plan.encode_values: x_local must be a CUDA tensor")
        want = torch.complex128 if self.dtype in ("complex128", "c128") else torch.complex64
        if x_local.dtype != want:
            raise InvalidArgument(f"Plan.encode_values: x_local must be {want}")
        xl = x_local.reshape(1, -1) if x_local.dim() == 1 else x_local
        if xl.stride(-1) != 1:
            raise InvalidArgument("Plan.encode_values: x_local rows must be contiguous")
        batch, span = int(xl.shape[0]), int(xl.shape[1])
        row_stride = span if batch == 1 else int(xl.stride(0))  # size-1 dims carry any stride
        seeds = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64).reshape(-1))
        if seeds.size != batch:
            raise InvalidArgument("Plan.encode_values: need one seed per signal")
        if y is None:
            y = torch.empty((batch, self.values_per_signal), dtype=torch.complex128,
                            device=xl.device)
        err = C.create_string_buffer(1024)
        status = self._lib.msfft_encode_values(
            self._h, batch, C.c_void_p(xl.data_ptr()), row_stride, int(x_lo),
            int(x_lo) + span, seeds.ctypes.data_as(C.POINTER(C.c_uint64)),
            C.c_void_p(y.data_ptr()), _L.MSFFT_FLAG_ASSUME_VALID if assume_valid else 0,
            C.c_void_p(_torch_stream(xl.device)), err, 1024)
        _raise(status, err)
        return y

    def encode_values_part(self, x, seeds, part: int, parts: int, y=None,
                           assume_valid: bool = False):
        """Tap-range sharding (x replicated: whole signals on this rank):
        PARTIAL bucket values from this part's share of every encode task's
        taps; the `parts` vectors sum to the full vector.  Per-rank encode
        work is 1/parts of the transform's.  Iterations with b > 256 are left
        as folds: decode the sum with decode_values(..., folds=True)."""
        import torch
        if not (_is_torch(x) and x.is_cuda):
            raise InvalidArgument("Plan.encode_values_part: x must be a CUDA tensor")
        want = torch.complex128 if self.dtype in ("complex128", "c128") else torch.complex64
        if x.dtype != want:
            raise InvalidArgument(f"Plan.encode_values_part: x must be {want}")
        xl = x.reshape(1, -1) if x.dim() == 1 else x
        if xl.stride(-1) != 1 or int(xl.shape[1]) != self.n:
            raise InvalidArgument("Plan.encode_values_part: x rows must be whole contiguous signals")
        batch = int(xl.shape[0])
        row_stride = self.n if batch == 1 else int(xl.stride(0))
        seeds = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64).reshape(-1))
        if seeds.size != batch:
            raise InvalidArgument("Plan.encode_values_part: need one seed per signal")
        if y is None:
            y = torch.empty((batch, self.values_per_signal), dtype=torch.complex128,
                            device=xl.device)
        err = C.create_string_buffer(1024)
        status = self._lib.msfft_encode_values_part(
            self._h, batch, C.c_void_p(xl.data_ptr()), row_stride, int(part), int(parts),
            seeds.ctypes.data_as(C.POINTER(C.c_uint64)), C.c_void_p(y.data_ptr()),
            _L.MSFFT_FLAG_ASSUME_VALID if assume_valid else 0,
            C.c_void_p(_torch_stream(xl.device)), err, 1024)
        _raise(status, err)
        return y

    def decode_values(self, y, seeds, out=None, folds: bool = False):
        """Selection / locate / estimate on summed bucket values y (consumed).
        folds=True: y is a sum of encode_values_part outputs, whose b > 256
        iterations are still folds (their FFTs run first, once).
        Returns (f, c, count) CUDA tensors ([B,k] int64, [B,k] complex128, [B])."""
        import torch
        if not (_is_torch(y) and y.is_cuda and y.dtype == torch.complex128 and y.is_contiguous()):
            raise InvalidArgument("Plan.decode_values: y must be a contiguous complex128 CUDA tensor")
        batch = int(y.numel() // self.values_per_signal)
        seeds = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64).reshape(-1))
        if seeds.size != batch:
            raise InvalidArgument("Plan.decode_values: need one seed per signal")
        if out is None:
            out = (torch.zeros((batch, self.k), dtype=torch.int64, device=y.device),
                   torch.zeros((batch, self.k), dtype=torch.complex128, device=y.device),
                   torch.zeros(batch, dtype=torch.int64, device=y.device))
        f, c, cnt = out
        err = C.create_string_buffer(1024)
        fn = self._lib.msfft_decode_folds if folds else self._lib.msfft_decode_values
        status = fn(
            self._h, batch, C.c_void_p(y.data_ptr()), seeds.ctypes.data_as(C.POINTER(C.c_uint64)),
            C.c_void_p(f.data_ptr()), C.c_void_p(c.data_ptr()), C.c_void_p(cnt.data_ptr()),
            C.c_void_p(_torch_stream(y.device)), err, 1024)
        _raise(status, err)
        return f, c, cnt


def window(n: int, b: int, delta: float, device: int = -1):
    """(w, taps) exactly as design_flat_window (proj/src/window.cpp:105-177)."""
    L = _L.lib()
    w = C.c_int64()
    err = C.create_string_buffer(1024)
    _raise(L.msfft_window(n, b, float(delta), device, C.byref(w), None, 0, err, 1024), err)
    taps = np.zeros(w.value, np.float64)
    _raise(L.msfft_window(n, b, float(delta), device, C.byref(w),
                          taps.ctypes.data_as(C.POINTER(C.c_double)), w.value, err, 1024), err)
    return w.value, taps


def window_response(n: int, b: int, delta: float, idx, device: int = -1) -> np.ndarray:
    """G_d from the device response table (FlatWindow::response_at)."""
    L = _L.lib()
    idx = np.ascontiguousarray(np.asarray(idx, dtype=np.int64))
    out = np.zeros(idx.size, np.float64)
    err = C.create_string_buffer(1024)
    _raise(L.msfft_window_response(n, b, float(delta), device,
                                   idx.ctypes.data_as(C.POINTER(C.c_int64)), idx.size,
                                   out.ctypes.data_as(C.POINTER(C.c_double)), err, 1024), err)
    return out


def trace(x, k: int, cfg: MultiscaleConfig | None = None, seed: int = 0, delta: float = 1e-8,
          values_per_signal: int = 0, selections: int = 0):
    """Kernel-level view of one transform: every iteration's bucket vectors
    before (encode output) and after the subtraction of known tones, the
    per-rank selection results (bucket, f or -1, value) and the final
    spectrum.  values_per_signal = sum_m rounds_m*b_m and selections =
    sum_m min(k_m, b_m) size the buffers (both follow from the plan)."""
    cfg = cfg or MultiscaleConfig()
    L = _L.lib()
    a = np.asarray(x)
    dt = _L.MSFFT_C64 if a.dtype == np.complex64 else _L.MSFFT_C128
    a = np.ascontiguousarray(a if dt == _L.MSFFT_C64 else a.astype(np.complex128))
    n = a.shape[-1]
    pre = np.zeros(2 * values_per_signal, np.float64)
    post = np.zeros(2 * values_per_signal, np.float64)
    sb = np.full(max(selections, 1), -2, np.int64)
    sf = np.full(max(selections, 1), -2, np.int64)
    sv = np.zeros(2 * max(selections, 1), np.float64)
    cap = max(int(k), 1)
    f = np.zeros(cap, np.int64)
    c = np.zeros(2 * cap, np.float64)
    cnt = C.c_int64()
    err = C.create_string_buffer(1024)
    PD = C.POINTER(C.c_double)
    PI = C.POINTER(C.c_int64)
    _raise(L.msfft_trace(C.c_void_p(a.ctypes.data), n, dt, int(k), int(cfg.l), float(cfg.q),
                         int(seed) & ((1 << 64) - 1), float(delta), pre.ctypes.data_as(PD),
                         post.ctypes.data_as(PD), sb.ctypes.data_as(PI), sf.ctypes.data_as(PI),
                         sv.ctypes.data_as(PD), cap, f.ctypes.data_as(PI),
                         c.ctypes.data_as(PD), C.byref(cnt), err, 1024), err)
    m = cnt.value
    return dict(pre=pre.view(np.complex128), post=post.view(np.complex128),
                sel_bucket=sb[:selections], sel_f=sf[:selections],
                sel_value=sv.view(np.complex128)[:selections],
                f=f[:m].copy(), c=c.view(np.complex128)[:m].copy())
