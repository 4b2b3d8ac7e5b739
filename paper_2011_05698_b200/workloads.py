"""Seeded synthetic signals with the BASELINE.json configs' laws (harness, not
the hot path).

Each signal is x = IDFT of a K-sparse spectrum, with the reference's
unnormalised inverse convention x_j = sum_f c_f e^{+2 pi i j f / N}
(idft_dense, proj/src/signal.cpp:50-58), plus complex white Gaussian noise
scaled to the exact realised SNR as add_awgn does (signal.cpp:129-152).
The O(N log N) inverse FFT replaces the reference's O(N K) synthesize
(SURVEY.md section 8(d)); it runs on the GPU through torch (cuFFT is fine for
test-data generation -- it is never on the measured path).

Config laws (BASELINE.json "configs"):
  C1  N=2^16, K=50, |c|=1, exact                      -> use the reference's
      own generate_test_signal (oracle) so bytes match its harness;
  C2  N=2^20, K=100, |c|=1, 20 dB                      -> same;
  C3  N=2^24, K=1000, |c|~U[0.5,2], 30 dB, min separation 4N/B;
  C4  N=2^22, K=64, |c|=1, 25 dB, complex64, 1024 per-signal seeds;
  C5  N=2^27, K=10000, |c| log-uniform [0.1, 10], 20 dB.
"""
from __future__ import annotations

import math

import numpy as np

from . import splitmix64

C4 = dict(n=1 << 22, k=64, snr_db=25.0, batch=1024, dtype="complex64", delta=1e-6,
          magnitude="unit")


def signal_seed(base: int, index: int) -> int:
    return splitmix64((base + index) & ((1 << 64) - 1))


def algo_seed(sig_seed: int) -> int:
    """Algorithm seed as the reference bench derives it (bench.cpp:117)."""
    return splitmix64(sig_seed ^ 0x53)


def sparse_support(n: int, k: int, seed: int, magnitude: str = "unit", min_sep: int = 0):
    """(positions ascending, complex coefficients) for one signal."""
    rng = np.random.default_rng(seed)
    if min_sep > 0:
        # gap-shift construction: k gaps of at least min_sep summing to n
        slack = n - k * min_sep
        if slack < 0:
            raise ValueError("sparse_support: min separation too large")
        cuts = np.sort(rng.integers(0, slack + 1, size=k))
        start = int(rng.integers(0, n))
        pos = (start + cuts + np.arange(k) * min_sep) % n
        pos = np.sort(pos.astype(np.int64))
    else:
        pos = np.sort(rng.choice(n, size=k, replace=False).astype(np.int64))
    phase = rng.uniform(0.0, 2.0 * math.pi, size=k)
    if magnitude == "unit":
        mag = np.ones(k)
    elif magnitude == "uniform_0.5_2":
        mag = rng.uniform(0.5, 2.0, size=k)
    elif magnitude == "loguniform_0.1_10":
        mag = 10.0 ** rng.uniform(-1.0, 1.0, size=k)
    else:
        raise ValueError(magnitude)
    return pos, mag * np.exp(1j * phase)


def make_batch(n: int, k: int, seeds, snr_db: float | None, device, dtype="complex64",
               magnitude: str = "unit", min_sep: int = 0, chunk: int = 32):
    """torch tensor [len(seeds), n] of signals on `device` (generated in
    chunks); returns (x, truths) with truths a list of (positions, coeffs)."""
    import torch

    tdt = torch.complex64 if dtype == "complex64" else torch.complex128
    B = len(seeds)
    x = torch.empty((B, n), dtype=tdt, device=device)
    truths = []
    for c0 in range(0, B, chunk):
        c1 = min(B, c0 + chunk)
        spec = torch.zeros((c1 - c0, n), dtype=torch.complex128 if tdt == torch.complex128
                           else torch.complex64, device=device)
        for i in range(c0, c1):
            pos, coef = sparse_support(n, k, int(seeds[i]), magnitude, min_sep)
            truths.append((pos, coef))
            spec[i - c0, torch.as_tensor(pos, device=device)] = torch.as_tensor(
                coef, dtype=spec.dtype, device=device)
        xc = torch.fft.ifft(spec, dim=1) * n
        if snr_db is not None and math.isfinite(snr_db):
            g = torch.Generator(device=device)
            g.manual_seed(int(seeds[c0]) & ((1 << 63) - 1))
            noise = torch.randn((c1 - c0, n), dtype=xc.dtype, device=device, generator=g)
            ps = (xc.abs() ** 2).double().sum(dim=1)
            pn = (noise.abs() ** 2).double().sum(dim=1)
            scale = torch.sqrt(ps * 10.0 ** (-snr_db / 10.0) / pn).to(xc.real.dtype)
            xc = xc + noise * scale[:, None]
        x[c0:c1] = xc.to(tdt)
        del spec, xc
    return x, truths


def make_signal_np(n: int, k: int, seed: int, snr_db: float | None, dtype="complex128",
                   magnitude: str = "unit", min_sep: int = 0):
    """One signal with numpy only (pocketfft + PCG64): bit-reproducible on any
    host with this image, so golden fixtures can store the recipe instead of
    the samples.  Returns (x, positions, coeffs)."""
    pos, coef = sparse_support(n, k, seed, magnitude, min_sep)
    spec = np.zeros(n, np.complex128)
    spec[pos] = coef
    x = np.fft.ifft(spec) * n
    if snr_db is not None and math.isfinite(snr_db):
        rng = np.random.default_rng(splitmix64(seed ^ 0x52))
        noise = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        ps = float(np.sum(np.abs(x) ** 2))
        pn = float(np.sum(np.abs(noise) ** 2))
        x = x + math.sqrt(ps * 10.0 ** (-snr_db / 10.0) / pn) * noise
    return x.astype(np.complex64 if dtype == "complex64" else np.complex128), pos, coef
