"""The steps either side of the hot path, through
the C ABI: signal generation and noise on the device, dense DFT scoring, and
the reference's file formats.  Mirrors proj/include/msfft/signal.hpp and
io.hpp (names, argument meaning, exception types and messages).

Arrays may be numpy (host) or torch CUDA tensors (device); results come back
in the same place.  Complex64 inputs are accepted where the reference takes a
ComplexSignal (exact upcast); signal files always hold float64 pairs.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _lib as _L
from . import InvalidArgument, _is_torch, _raise

__all__ = ["EvalMetrics", "generate_test_signal", "synthesize", "add_awgn", "dft_dense",
           "idft_dense", "top_k_spectrum", "error_metrics", "read_signal_file",
           "write_signal_file", "read_truth_csv", "write_truth_csv", "signal_file_length",
           "PhaseErrorHistogram", "run_phase_experiment"]


@dataclass
class EvalMetrics:
    """signal.hpp:31-38 (runtime / sample fields are the caller's)."""
    l0_err: int = 0
    l1_err: float = 0.0
    l2_err: float = 0.0


def _err():
    return C.create_string_buffer(1024)


def _dtype_code(dtype) -> int:
    name = str(dtype).replace("torch.", "").replace("numpy.", "")
    if name in ("complex128", "c128"):
        return _L.MSFFT_C128
    if name in ("complex64", "c64"):
        return _L.MSFFT_C64
    raise InvalidArgument(f"unsupported dtype {dtype}")


def _buf(x):
    """-> (pointer, location, dtype code, keepalive) of a contiguous buffer."""
    if _is_torch(x):
        if not x.is_contiguous():
            raise InvalidArgument("tensor must be contiguous")
        return (C.c_void_p(x.data_ptr()), _L.MSFFT_DEVICE if x.is_cuda else _L.MSFFT_HOST,
                _dtype_code(x.dtype) if x.is_complex() else None, x)
    a = np.asarray(x)
    if not a.flags.c_contiguous:
        a = np.ascontiguousarray(a)
    code = _dtype_code(a.dtype) if np.iscomplexobj(a) else None
    return C.c_void_p(a.ctypes.data), _L.MSFFT_HOST, code, a


def _alloc(like, shape, complex_dtype):
    if _is_torch(like) and like.is_cuda:
        import torch
        return torch.empty(shape, dtype=getattr(torch, complex_dtype), device=like.device)
    return np.empty(shape, dtype=complex_dtype)


def _spec_arrays(f, c):
    f = np.ascontiguousarray(np.asarray(f, dtype=np.int64).reshape(-1))
    c = np.ascontiguousarray(np.asarray(c, dtype=np.complex128).reshape(-1))
    if f.size != c.size:
        raise InvalidArgument("positions and coefficients differ in length")
    return f, c


def generate_test_signal(n: int, k: int, seed: int, dtype: str = "complex128", device=None):
    """generate_test_signal (signal.cpp:116-121) -> (x, truth_f, truth_c,
    bit_exact).  device: None for a numpy result, else a torch device (CUDA).
    The truth is the reference's draw; x is synthesized on the GPU."""
    x = _target(n, dtype, device)
    f = np.zeros(max(k, 1), np.int64)
    c = np.zeros(max(k, 1), np.complex128)
    exact = C.c_int32()
    ptr, loc, _, _ = _buf(x)
    e = _err()
    _raise(_L.lib().msfft_generate_test_signal(int(n), int(k), int(seed) & (2**64 - 1),
                                               _dtype_code(dtype), loc, ptr,
                                               C.c_void_p(f.ctypes.data),
                                               C.c_void_p(c.ctypes.data), C.byref(exact), e,
                                               1024), e)
    return x, f[:k], c[:k], bool(exact.value)


def _target(n, dtype, device):
    if device is None:
        return np.zeros(int(n), dtype=dtype)
    import torch
    return torch.zeros(int(n), dtype=getattr(torch, dtype), device=device)


def synthesize(n: int, f, c, dtype: str = "complex128", device=None):
    """synthesize (signal.cpp:76-98) -> (x, bit_exact)."""
    f, c = _spec_arrays(f, c)
    x = _target(n, dtype, device)
    ptr, loc, _, _ = _buf(x)
    exact = C.c_int32()
    e = _err()
    _raise(_L.lib().msfft_synthesize(int(n), C.c_void_p(f.ctypes.data), C.c_void_p(c.ctypes.data),
                                     f.size, _dtype_code(dtype), loc, ptr, C.byref(exact), e,
                                     1024), e)
    return x, bool(exact.value)


def add_awgn(x, snr_db: float, seed: int):
    """add_awgn (signal.cpp:123-152): returns a noisy copy of x (same place,
    same dtype).  Noise: Philox-based Box-Muller on the device."""
    y = x.clone() if _is_torch(x) else np.array(x, copy=True)
    ptr, loc, code, keep = _buf(y)
    if code is None:
        raise InvalidArgument("add_awgn: x must be complex")
    e = _err()
    _raise(_L.lib().msfft_add_awgn(ptr, int(keep.shape[-1]), code, loc, float(snr_db),
                                   int(seed) & (2**64 - 1), e, 1024), e)
    return y


def dft_dense(x):
    """dft_dense (signal.cpp:37-44) of one signal or a (batch, n) stack."""
    ptr, loc, code, keep = _buf(x)
    if code is None:
        raise InvalidArgument("dft_dense: x must be complex")
    n = int(keep.shape[-1])
    batch = int(np.prod(keep.shape[:-1])) if len(keep.shape) > 1 else 1
    out = _alloc(keep, tuple(keep.shape), "complex128")
    optr, _, _, _ = _buf(out)
    e = _err()
    _raise(_L.lib().msfft_dft_dense(ptr, n, batch, code, loc, optr, e, 1024), e)
    return out


def idft_dense(spec):
    """idft_dense (signal.cpp:46-54): the unnormalised inverse."""
    if _is_torch(spec):
        import torch
        spec = spec.to(torch.complex128).contiguous()
    else:
        spec = np.ascontiguousarray(np.asarray(spec, dtype=np.complex128))
    ptr, loc, _, keep = _buf(spec)
    n = int(keep.shape[-1])
    batch = int(np.prod(keep.shape[:-1])) if len(keep.shape) > 1 else 1
    out = _alloc(keep, tuple(keep.shape), "complex128")
    optr, _, _, _ = _buf(out)
    e = _err()
    _raise(_L.lib().msfft_idft_dense(ptr, n, batch, loc, optr, e, 1024), e)
    return out


def top_k_spectrum(spec, k: int):
    """top_k_spectrum (bench.cpp:33-46) -> (f ascending, c) numpy arrays."""
    if _is_torch(spec):
        import torch
        spec = spec.to(torch.complex128).contiguous()
    else:
        spec = np.ascontiguousarray(np.asarray(spec, dtype=np.complex128))
    ptr, loc, _, keep = _buf(spec)
    n = int(keep.shape[-1])
    cap = max(min(int(k), n), 1)
    f = np.zeros(cap, np.int64)
    c = np.zeros(cap, np.complex128)
    cnt = C.c_int64()
    e = _err()
    _raise(_L.lib().msfft_top_k_spectrum(ptr, n, int(k), loc, C.c_void_p(f.ctypes.data),
                                         C.c_void_p(c.ctypes.data), C.byref(cnt), e, 1024), e)
    return f[:cnt.value], c[:cnt.value]


def error_metrics(truth_n: int, truth_f, truth_c, est_n: int, est_f, est_c, k: int) -> EvalMetrics:
    """error_metrics (signal.cpp:154-184) over (f, c) lists."""
    tf, tc = _spec_arrays(truth_f, truth_c)
    ef, ec = _spec_arrays(est_f, est_c)
    m = _L.EvalMetricsC()
    e = _err()
    _raise(_L.lib().msfft_error_metrics(int(truth_n), C.c_void_p(tf.ctypes.data),
                                        C.c_void_p(tc.ctypes.data), tf.size, int(est_n),
                                        C.c_void_p(ef.ctypes.data), C.c_void_p(ec.ctypes.data),
                                        ef.size, int(k), C.byref(m), e, 1024), e)
    return EvalMetrics(int(m.l0_err), float(m.l1_err), float(m.l2_err))


def signal_file_length(path) -> int:
    n = C.c_int64()
    e = _err()
    _raise(_L.lib().msfft_signal_file_length(os.fsencode(path), C.byref(n), e, 1024), e)
    return n.value


def read_signal_file(path, dtype: str = "complex128", device=None):
    """read_signal_file (io.cpp:30-55) into numpy (device None) or a torch
    CUDA tensor."""
    n = signal_file_length(path)
    x = _target(n, dtype, device)
    ptr, loc, _, _ = _buf(x)
    got = C.c_int64()
    e = _err()
    _raise(_L.lib().msfft_read_signal_file(os.fsencode(path), _dtype_code(dtype), loc, ptr, n,
                                           C.byref(got), e, 1024), e)
    return x


def write_signal_file(path, x) -> None:
    """write_signal_file (io.cpp:17-28) from numpy or a torch tensor."""
    ptr, loc, code, keep = _buf(x)
    if code is None:
        raise InvalidArgument("write_signal_file: x must be complex")
    e = _err()
    _raise(_L.lib().msfft_write_signal_file(os.fsencode(path), ptr, int(keep.shape[-1]), code,
                                            loc, e, 1024), e)


def write_truth_csv(path, f, c) -> None:
    """write_truth_csv (io.cpp:57-68)."""
    f, c = _spec_arrays(f, c)
    e = _err()
    _raise(_L.lib().msfft_write_truth_csv(os.fsencode(path), C.c_void_p(f.ctypes.data),
                                          C.c_void_p(c.ctypes.data), f.size, e, 1024), e)


def read_truth_csv(path, n: int):
    """read_truth_csv (io.cpp:70-92) -> (f ascending, c)."""
    cap = 1 << 16
    while True:
        f = np.zeros(cap, np.int64)
        c = np.zeros(cap, np.complex128)
        cnt = C.c_int64()
        e = _err()
        _raise(_L.lib().msfft_read_truth_csv(os.fsencode(path), int(n), C.c_void_p(f.ctypes.data),
                                             C.c_void_p(c.ctypes.data), cap, C.byref(cnt), e,
                                             1024), e)
        if cnt.value <= cap:
            return f[:cnt.value], c[:cnt.value]
        cap = cnt.value


@dataclass
class PhaseErrorHistogram:
    """phase_mc.hpp:19-30."""
    snr_db: float
    n: int
    k: int
    l_width: int
    trials: int
    bin_mass: np.ndarray
    p50: float
    p99: float
    max: float
    samples: np.ndarray | None = None  # accepted dphi in acceptance order (if requested)

    kBinLo = -6.0
    kBinWidth = 0.1
    kBinCount = 70

    @staticmethod
    def bin_center(i: int) -> float:
        return -6.0 + 0.1 * (i + 0.5)


def run_phase_experiment(n: int, k: int, b: int, snr_list, trials: int, seed: int,
                         keep_trials: bool = False):
    """run_phase_experiment (phase_mc.cpp:166-212) on the GPU -> list of
    PhaseErrorHistogram; with keep_trials, also a list (per SNR) of structured
    trial records (dphi, u, bucket, tau, y0, y_tau, measured_phi, true_phi)."""
    snr = np.ascontiguousarray(np.asarray(list(snr_list), dtype=np.float64))
    hs = (_L.PhaseHistogramC * max(snr.size, 1))()
    tr = (_L.PhaseTrialC * (snr.size * int(trials)))() if keep_trials and trials > 0 else None
    e = _err()
    _raise(_L.lib().msfft_phase_experiment(int(n), int(k), int(b), C.c_void_p(snr.ctypes.data),
                                           snr.size, int(trials), int(seed) & (2**64 - 1), hs,
                                           tr, e, 1024), e)
    out, trials_out = [], []
    for i in range(snr.size):
        h = hs[i]
        out.append(PhaseErrorHistogram(h.snr_db, h.n, h.k, h.l_width, h.trials,
                                       np.array(h.bin_mass[:]), h.p50, h.p99, h.max))
        if tr is not None:
            rows = [tr[i * trials + t] for t in range(trials)]
            trials_out.append([{"dphi": r.dphi, "u": r.u, "bucket": r.bucket, "tau": r.tau,
                                "y0": complex(r.y0[0], r.y0[1]),
                                "y_tau": complex(r.y_tau[0], r.y_tau[1]),
                                "measured_phi": r.measured_phi, "true_phi": r.true_phi}
                               for r in rows])
            out[-1].samples = np.array([r["dphi"] for r in trials_out[-1]])
    return (out, trials_out) if keep_trials else out
