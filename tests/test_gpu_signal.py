"""SURVEY 8(f) rows 2-3 on the device: generate_test_signal / synthesize,
add_awgn, dft_dense / idft_dense, top_k_spectrum -- against the reference's
own signal.cpp / bench.cpp (oracle), bit-exact where the reference's
arithmetic is reproducible, else with the stated tolerance."""
import numpy as np
import pytest

import paper_2011_05698_b200 as M
import paper_2011_05698_b200.signal as S

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,k,seed", [(8192, 50, 11), (1 << 16, 50, 3), (1 << 20, 100, 7),
                                      (512, 3, 1), (64, 64, 2), (16, 1, 4)])
def test_generate_test_signal_bit_exact(oracle, n, k, seed):
    x, f, c, exact = S.generate_test_signal(n, k, seed)
    rx, rf, rc = oracle.generate_test_signal(n, k, seed)
    assert exact
    assert np.array_equal(f, rf) and np.array_equal(c, rc)
    assert np.array_equal(x, rx)


def test_generate_on_device_and_complex64(oracle):
    import torch
    x, f, c, exact = S.generate_test_signal(1 << 14, 40, 9, "complex128", "cuda")
    rx, _, _ = oracle.generate_test_signal(1 << 14, 40, 9)
    assert x.is_cuda and exact and np.array_equal(x.cpu().numpy(), rx)
    x64, _, _, _ = S.generate_test_signal(1 << 14, 40, 9, "complex64", "cuda")
    assert x64.dtype == torch.complex64
    assert np.array_equal(x64.cpu().numpy(), rx.astype(np.complex64))


def test_synthesize_edge_cases(oracle):
    x, _ = S.synthesize(128, [], [])
    assert not np.any(x)
    x, _ = S.synthesize(128, [0], [1.0])
    assert np.max(np.abs(x - 1)) < 1e-12
    f = [3, 900, 2000]
    c = [1 + 1j, -0.5, 2j]
    x, exact = S.synthesize(4096, f, c)
    assert exact and np.array_equal(x, oracle.synthesize(4096, f, c))
    with pytest.raises(M.InvalidArgument, match="SparseSpectrum: position out of range"):
        S.synthesize(64, [64], [1])
    with pytest.raises(M.InvalidArgument, match="SparseSpectrum: non-finite coefficient"):
        S.synthesize(64, [1], [np.nan])
    with pytest.raises(M.InvalidArgument, match="SparseSpectrum: n must be a power of two"):
        S.synthesize(48, [1], [1])
    with pytest.raises(M.InvalidArgument, match="random_sparse_spectrum: k out of range"):
        S.generate_test_signal(64, 65, 1)


def test_synthesize_large_table_fallback(oracle):
    """Beyond the 2^23-entry seed table the seeds come from device sincos:
    ulp-level agreement."""
    n, k = 1 << 20, 8200  # 8200 * 1024 blocks > 2^23
    rng = np.random.default_rng(0)
    f = np.sort(rng.choice(n, k, replace=False))
    c = np.exp(2j * np.pi * rng.random(k))
    x, exact = S.synthesize(n, f, c, "complex128", "cuda")
    assert not exact
    ref = oracle.synthesize(n, f, c)
    err = np.max(np.abs(x.cpu().numpy() - ref)) / np.max(np.abs(ref))
    assert err < 1e-12, err


def test_add_awgn_power_and_rules():
    import torch
    x, f, c, _ = S.generate_test_signal(8192, 50, 21)
    sig = np.sum(np.abs(x) ** 2)
    for snr in (0.0, 20.0, 35.5):
        y = S.add_awgn(x, snr, 13)
        noise = np.sum(np.abs(y - x) ** 2)
        assert abs(noise / sig / 10 ** (-snr / 10) - 1) < 1e-9  # realised ratio = request
    assert np.array_equal(S.add_awgn(x, np.inf, 1), x)
    for bad in (np.nan, -np.inf):
        with pytest.raises(M.InvalidArgument, match="add_awgn: snr_db must be finite or \\+infinity"):
            S.add_awgn(x, bad, 1)
    xb = x.copy()
    xb[5] = np.inf
    with pytest.raises(M.InvalidArgument, match="ComplexSignal: non-finite sample"):
        S.add_awgn(xb, 10.0, 1)
    # deterministic per seed, different across seeds, same on host and device
    a, b = S.add_awgn(x, 10.0, 5), S.add_awgn(x, 10.0, 6)
    assert np.array_equal(a, S.add_awgn(x, 10.0, 5)) and not np.array_equal(a, b)
    xd = torch.as_tensor(x).cuda()
    assert np.array_equal(S.add_awgn(xd, 10.0, 5).cpu().numpy(), a)
    # the noise is standard complex Gaussian
    z = S.add_awgn(np.zeros(1 << 20, np.complex128) + 1.0, 0.0, 8) - 1.0
    g = np.concatenate([z.real, z.imag]) / np.sqrt(np.mean(np.abs(z) ** 2) / 2)
    assert abs(np.mean(g)) < 5e-3 and abs(np.mean(g ** 2) - 1) < 5e-3
    assert abs(np.mean(g ** 4) - 3) < 3e-2  # Gaussian kurtosis


@pytest.mark.parametrize("n", [64, 4096, 1 << 16, 1 << 20])
def test_dft_dense_bit_exact(oracle, n):
    rng = np.random.default_rng(n)
    x = rng.random(n) - 0.5 + 1j * (rng.random(n) - 0.5)
    X = S.dft_dense(x)
    assert np.array_equal(X, oracle.dft_dense(x))
    assert np.array_equal(S.idft_dense(X), oracle.idft_dense(X))


def test_dft_dense_batch_device_c64(oracle):
    import torch
    rng = np.random.default_rng(2)
    xs = (rng.standard_normal((3, 2048)) + 1j * rng.standard_normal((3, 2048))).astype(np.complex64)
    Xd = S.dft_dense(torch.as_tensor(xs).cuda())
    assert Xd.is_cuda and Xd.dtype == torch.complex128
    for i in range(3):
        assert np.array_equal(Xd[i].cpu().numpy(), oracle.dft_dense(xs[i].astype(np.complex128)))
    impulse = np.zeros(64, np.complex128)
    impulse[0] = 1
    assert np.all(S.dft_dense(impulse) == 1 / 64)
    with pytest.raises(M.InvalidArgument, match="ComplexSignal: non-finite sample"):
        S.dft_dense(np.full(64, np.nan, np.complex128))
    with pytest.raises(M.InvalidArgument, match="ComplexSignal: n must be a power of two >= 4"):
        S.dft_dense(np.zeros(48, np.complex128))
    with pytest.raises(M.InvalidArgument, match="idft_dense: size must be a power of two >= 4"):
        S.idft_dense(np.zeros(48, np.complex128))


def test_top_k_matches_reference(oracle):
    rng = np.random.default_rng(5)
    for n, k in ((4096, 20), (1 << 20, 1000), (1 << 16, 1), (256, 256), (256, 300)):
        spec = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        f, c = S.top_k_spectrum(spec, k)
        rf, rc = oracle.top_k_spectrum(spec, k)
        assert np.array_equal(f, rf) and np.array_equal(c, rc)
    # the dense scoring path of bench.cpp:131-137 end to end
    x, tf, tc, _ = S.generate_test_signal(8192, 50, 11)
    f, c = S.top_k_spectrum(S.dft_dense(x), 50)
    m = S.error_metrics(8192, tf, tc, 8192, f, c, 50)
    assert m.l0_err == 0 and m.l1_err < 1e-12
    # ties at the k-th magnitude keep the lowest indices
    spec = np.zeros(64, np.complex128)
    spec[[3, 10, 20, 40]] = [2, 1, 1j, -1]
    f, _ = S.top_k_spectrum(spec, 3)
    assert list(f) == [3, 10, 20]
    assert len(S.top_k_spectrum(spec, 0)[0]) == 0
