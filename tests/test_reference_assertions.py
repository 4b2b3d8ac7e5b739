"""The reference's own unit-test assertions (proj/tests/test_bucketizer.cpp,
test_flat_window.cpp), re-expressed in pytest against the CPU oracle --
doctest.h is absent, so the C++ tests cannot be compiled.
CPU only."""
import math

import numpy as np
import pytest

from conftest import oracle_kinds

KINDS = oracle_kinds()
pytestmark = pytest.mark.skipif(not KINDS, reason="no oracle library built")
TWO_PI = 2.0 * math.pi


@pytest.fixture(params=KINDS, scope="module")
def orc(request):
    from oracle import load
    return load(request.param)


def random_signal(n, seed):
    """test_bucketizer.cpp:26-33 analogue (uniform in [-0.5, 0.5))."""
    rng = np.random.default_rng(seed)
    return (rng.random(n) - 0.5) + 1j * (rng.random(n) - 0.5)


def matrix_pipeline(x, taps, b, sigma, tau):
    """Literal F_B U_L Q_L S_tau P_sigma x (test_bucketizer.cpp:38-69)."""
    n = x.size
    j = np.arange(n)
    v1 = x[(sigma * j) % n]
    v2 = v1[(j - tau) % n]
    w = taps.size
    h = (w - 1) // 2
    g = np.zeros(n)
    g[0] = taps[h]
    t = np.arange(1, h + 1)
    g[t] = taps[h + t]
    g[n - t] = taps[h - t]
    v2 = v2 * g
    v3 = np.zeros(b, np.complex128)
    np.add.at(v3, j % b, v2)
    k = np.arange(b)
    F = np.exp(-2j * np.pi * np.outer(k, k) / b)
    return F @ v3 / n


def test_mod_inverse(orc):
    assert orc.mod_inverse(1, 64) == 1
    assert orc.mod_inverse(3, 8) == 3
    assert orc.mod_inverse(5, 16) == 13
    for s in range(1, 256, 2):
        assert (s * orc.mod_inverse(s, 256)) % 256 == 1
    from oracle import OracleError
    with pytest.raises(OracleError):
        orc.mod_inverse(4, 16)


def test_random_params_uniform(orc):
    s, si = orc.random_params(1024, 123, 10000)
    assert np.all(s % 2 == 1)
    assert np.all((s * si) % 1024 == 1)
    counts = np.bincount((s - 1) // 2, minlength=512)
    expected = 10000 / 512
    chi2 = float(np.sum((counts - expected) ** 2 / expected))
    assert chi2 < 588.4  # 99th percentile, 511 dof
    a, _ = orc.random_params(1024, 99, 1)
    b, _ = orc.random_params(1024, 99, 1)
    assert a[0] == b[0]


def test_bucketize_zero_signal(orc):
    y = orc.bucketize(np.zeros(1024, np.complex128), 32, 1e-6, 77, 0)
    assert np.all(y == 0)


def test_matrix_pipeline_geometry_64_8_is_infeasible(orc):
    """test_bucketizer.cpp:128 lists (n, b) = (64, 8), (256, 16), (1024, 32)
    at delta 1e-6, but the reference's own designer rejects the first two
    windows, so those cases of the reference test throw instead of comparing
    (recorded in DESIGN.md).  (1024, 32) plus two extra feasible geometries
    are compared below."""
    from oracle import OracleError
    for n, b in ((64, 8), (256, 16)):
        with pytest.raises(OracleError) as ei:
            orc.window(n, b, 1e-6, taps=False)
        assert "no support w <= n-1 passes the band check" in str(ei.value)


@pytest.mark.parametrize("n,b", [(512, 16), (1024, 32), (2048, 32)])
def test_bucketize_equals_matrix_pipeline(orc, n, b):
    _, taps = orc.window(n, b, 1e-6)
    sig, _ = orc.random_params(n, 1000 + n, 20)
    rng = np.random.default_rng(n)
    for trial in range(20):
        x = random_signal(n, 500 + trial)
        tau = int(rng.integers(0, n))
        fast = orc.bucketize(x, b, 1e-6, int(sig[trial]), tau)
        slow = matrix_pipeline(x, taps, b, int(sig[trial]), tau)
        assert np.max(np.abs(fast - slow)) < 1e-9


def test_single_tone_bucket_energy(orc):
    n, b = 8192, 256
    L = n // b
    for f in (100, 5000, 8191, 16, 48):
        spec = np.zeros(n, np.complex128)
        spec[f] = 0.8 + 0.6j
        x = np.fft.ifft(spec) * n
        y = orc.bucketize(x, b, 1e-6, 1, 0)
        i = orc.bucket_of(f, L, b)
        assert abs(y[i]) >= (1.0 - 1e-6) - 1e-9
        for j in range(b):
            dist = min((j - i) % b, (i - j) % b)
            if dist >= 2:
                assert abs(y[j]) <= 1e-6 + 1e-9


def test_predict_matches_bucketize(orc):
    n, b, delta = 8192, 256, 1e-6
    rng = np.random.default_rng(31)
    sig, _ = orc.random_params(n, 31, 5)
    for trial in range(5):
        f = int(rng.integers(0, n))
        c = np.exp(1j * TWO_PI * rng.random())
        spec = np.zeros(n, np.complex128)
        spec[f] = c
        x = np.fft.ifft(spec) * n
        tau = int(rng.integers(0, n))
        real = orc.bucketize(x, b, delta, int(sig[trial]), tau)
        pred = orc.predict(n, b, delta, [f], [c], int(sig[trial]), tau)
        assert np.max(np.abs(real - pred)) <= 5 * delta


def test_predict_k50_within_250_delta(orc):
    n, b, delta = 8192, 256, 1e-6
    rng = np.random.default_rng(77)
    f = np.sort(rng.choice(n, 50, replace=False))
    c = np.exp(1j * TWO_PI * rng.random(50))
    spec = np.zeros(n, np.complex128)
    spec[f] = c
    x = np.fft.ifft(spec) * n
    sig, _ = orc.random_params(n, 77, 1)
    real = orc.bucketize(x, b, delta, int(sig[0]), 123)
    pred = orc.predict(n, b, delta, f, c, int(sig[0]), 123)
    assert np.max(np.abs(real - pred)) <= 50 * 5 * delta


def test_predict_empty(orc):
    pred = orc.predict(1024, 32, 1e-6, [], np.zeros(0, np.complex128), 5, 0)
    assert np.all(pred == 0)


def test_permutation_law():
    """Eq. 8: DFT of x_{sigma(j - tau)} at sigma*i is X_i w^{sigma tau i}."""
    n = 256
    x = random_signal(n, 9)
    sigma, tau = 77, 13
    j = np.arange(n)
    xp = x[(sigma * ((j - tau) % n)) % n]
    spec, spec_p = np.fft.fft(x) / n, np.fft.fft(xp) / n
    want = spec * np.exp(-2j * np.pi * ((sigma * tau * j) % n) / n)
    assert np.max(np.abs(spec_p[(sigma * j) % n] - want)) < 1e-9


def test_index_map_bijection(orc):
    n = 4096
    s, _ = orc.random_params(n, 17, 1)
    tau = 1234
    idx = (int(s[0]) * ((np.arange(n) - tau) % n)) % n
    assert np.unique(idx).size == n


def test_bucket_of_rounding(orc):
    assert orc.bucket_of(16, 32, 256) == 1
    assert orc.bucket_of(15, 32, 256) == 0
    assert orc.bucket_of(8192 - 16, 32, 256) == 0
    assert orc.bucket_of(8192 - 17, 32, 256) == 255


def padded_response(n, taps):
    w = taps.size
    h = (w - 1) // 2
    p = np.zeros(n, np.complex128)
    p[0] = taps[h]
    t = np.arange(1, h + 1)
    p[t] = taps[h + t]
    p[n - t] = taps[h - t]
    return np.fft.fft(p) / n


@pytest.mark.parametrize("n,b,delta", [(8192, 64, 1e-8), (8192, 256, 1e-6), (16384, 128, 1e-8)])
def test_window_three_bands(orc, n, b, delta):
    w, taps = orc.window(n, b, delta)
    L = n // b
    mag = np.abs(padded_response(n, taps))
    d = np.minimum(np.arange(n), n - np.arange(n))
    tol = 1e-12  # numpy's FFT vs the reference's radix-2: rounding only
    assert np.all(np.abs(mag[d <= L // 2] - 1.0) <= delta + tol)
    assert np.all(mag[d >= L] <= delta + tol)
    assert np.all(mag[(d > L // 2) & (d < L)] <= 1.0 + delta + tol)


def test_window_symmetry_and_response(orc):
    n, b = 4096, 64
    w, taps = orc.window(n, b, 1e-6)
    h = (w - 1) // 2
    assert w % 2 == 1
    assert np.allclose(taps[h:], taps[h::-1], rtol=1e-14, atol=0)
    for i in (1, 5, 17, 100, 2000):
        r = orc.response_at(n, b, 1e-6, [i, -i, i + n])
        assert abs(r[0] - r[1]) <= 1e-12 * max(1.0, abs(r[0]))
        assert abs(r[0] - r[2]) <= 1e-12 * max(1.0, abs(r[0]))
    w2, taps2 = orc.window(4096, 64, 1e-8)
    resp = padded_response(4096, taps2)
    idx = np.random.default_rng(123).integers(0, 4096, 250)
    assert np.max(np.abs(orc.response_at(4096, 64, 1e-8, idx) - resp[idx])) < 1e-10


def test_window_support_ratio(orc):
    w256, _ = orc.window(65536, 256, 1e-6, taps=False)
    w512, _ = orc.window(65536, 512, 1e-6, taps=False)
    assert 1.7 <= w512 / w256 <= 2.3


def test_window_parameter_errors(orc):
    from oracle import OracleError
    for args in ((8192, 256, 1e-8), (8192, 2048, 1e-6), (8192, 3, 1e-6), (8192, 64, 0.5),
                 (8192, 64, 0.0), (1000, 10, 1e-6)):
        with pytest.raises(OracleError) as ei:
            orc.window(*args, taps=False)
        assert ei.value.kind == "invalid_argument"
