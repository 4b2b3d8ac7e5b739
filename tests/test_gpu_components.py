"""The component API (bucketize, predict_buckets, subtract,
locate_frequency, estimate_value) on the GPU against the compiled reference,
and a whole sfft4 composed from those components in the reference's order
(sfft4.cpp:38-187) against the fused GPU transform and the reference."""
import math

import numpy as np
import pytest

import paper_2011_05698_b200 as M
from paper_2011_05698_b200 import components as CMP
from helpers import assert_parity, make_signal

pytestmark = pytest.mark.gpu


def _odd_sigmas(n, count, seed):
    rng = np.random.default_rng(seed)
    return [int(2 * rng.integers(0, n // 2) + 1) for _ in range(count)]


@pytest.mark.parametrize("n,b,delta,dtype", [(1 << 14, 64, 1e-8, "complex128"),
                                             (1 << 16, 256, 1e-6, "complex64"),
                                             (1 << 16, 2048, 1e-8, "complex128"),
                                             (1 << 18, 8192, 1e-6, "complex128")])
def test_bucketize_bit_identical(oracle, n, b, delta, dtype):
    """bucketize (bucketize.hpp:63-86): fold in ascending t, radix-2 DIT, /n --
    equal to the reference bit for bit, for several (sigma, tau) at once."""
    x = make_signal(oracle, dict(gen="np", n=n, k=20, seed=n + b, snr=20.0, dtype=dtype))
    win = CMP.flat_window(n, b, delta)
    rng = np.random.default_rng(b)
    params = [CMP.PermutationParams(s, 0, int(rng.integers(0, n)))
              for s in _odd_sigmas(n, 5, n ^ b)]
    params[0] = CMP.PermutationParams(params[0].sigma, 0, 0)
    sets = CMP.bucketize_rounds(x, win, params)
    for p, s in zip(params, sets):
        ref = oracle.bucketize(x.astype(np.complex128), b, delta, p.sigma, p.tau)
        assert np.array_equal(s.values, ref)
        assert s.samples_read == win.w and s.params == p


def test_bucketize_device_input(oracle):
    import torch
    n, b, delta = 1 << 15, 128, 1e-8
    x = make_signal(oracle, dict(gen="np", n=n, k=10, seed=3, snr=None, dtype="complex64"))
    win = CMP.flat_window(n, b, delta)
    p = CMP.PermutationParams(12345, 0, 777)
    host = CMP.bucketize(x, win, p)
    dev = CMP.bucketize(torch.as_tensor(x).cuda(), win, p)
    assert np.array_equal(host.values, dev.values)


def test_predict_buckets_matches_reference(oracle):
    """predict_buckets (bucketize.cpp:70-95): every known tone into its
    bucket and both neighbours, ascending f; G from the device table and the
    rotation by sincos, so ulp-level against libm."""
    n, b, delta = 1 << 16, 256, 1e-8
    rng = np.random.default_rng(9)
    f = np.sort(rng.choice(n, 60, replace=False)).astype(np.int64)
    c = np.exp(2j * np.pi * rng.random(60)) * (0.5 + rng.random(60))
    win = CMP.flat_window(n, b, delta)
    params = [CMP.PermutationParams(s, 0, int(rng.integers(0, n))) for s in _odd_sigmas(n, 4, 9)]
    got = CMP.predict_buckets(M.SparseSpectrum(n, f, c), win, params)
    for p, s in zip(params, got):
        ref = oracle.predict(n, b, delta, f, c, p.sigma, p.tau)
        assert np.max(np.abs(s.values - ref)) <= 1e-13 * np.max(np.abs(ref))


def test_predict_matches_bucketize_on_gpu(oracle):
    """test_bucketizer.cpp:165-199 re-expressed on the GPU components: a
    one-tone signal's buckets equal the prediction within 5 delta."""
    n, b, delta = 8192, 256, 1e-6
    rng = np.random.default_rng(31)
    win = CMP.flat_window(n, b, delta)
    for s in _odd_sigmas(n, 5, 31):
        fr = int(rng.integers(0, n))
        c = np.exp(2j * np.pi * rng.random())
        spec = np.zeros(n, np.complex128)
        spec[fr] = c
        x = np.fft.ifft(spec) * n
        p = CMP.PermutationParams(s, 0, int(rng.integers(0, n)))
        real = CMP.bucketize(x, win, p)
        pred = CMP.predict_buckets(M.SparseSpectrum(n, np.array([fr]), np.array([c])), win, p)
        assert np.max(np.abs(CMP.subtract(real, pred).values)) <= 5 * delta


def test_subtract_checks_geometry():
    p = CMP.PermutationParams(3, 0, 5)
    a = CMP.BucketSet(64, 8, np.ones(8, complex), p)
    with pytest.raises(M.InvalidArgument, match="subtract: bucket sets are not from the same round"):
        CMP.subtract(a, CMP.BucketSet(64, 8, np.ones(8, complex), CMP.PermutationParams(3, 0, 6)))
    assert np.array_equal(CMP.subtract(a, a).values, np.zeros(8, complex))


@pytest.mark.parametrize("n,b,l,q", [(1 << 14, 64, 16, 1.0), (1 << 16, 256, 8, 2.0),
                                     (1 << 16, 32, 4, 1.0)])
def test_locate_frequency_matches_reference(oracle, n, b, l, q):
    """locate_frequency (locate.cpp:83-123) for every bucket of a noisy
    multi-tone round set: identical u, stage count and nullopt cases."""
    delta = 1e-6
    cfg = M.MultiscaleConfig(l, q)
    x = make_signal(oracle, dict(gen="np", n=n, k=b // 4, seed=l, snr=15.0))
    win = CMP.flat_window(n, b, delta)
    taus = CMP.tau_plan(n // b, n, cfg)
    sg = _odd_sigmas(n, 1, n + l)[0]
    rounds = CMP.bucketize_rounds(x, win, [CMP.PermutationParams(sg, 0, t) for t in taus])
    rounds[1].values[3] = 0.0  # a zero round value: nullopt
    rounds[0].values[5] = 0.0  # a zero y0: nullopt
    got = CMP.locate_frequencies(range(b), rounds, cfg, win)
    vals = np.stack([r.values for r in rounds])
    for bucket in range(b):
        u, st = oracle.locate(n, b, delta, l, q, bucket, taus, vals)
        if u is None:
            assert got[bucket] is None, bucket
        else:
            assert got[bucket] == CMP.LocateOutcome(u, st), bucket
    assert got[3] is None and got[5] is None


def test_locate_frequency_errors():
    n, b = 1 << 12, 64
    win = CMP.FlatWindow(n, b, 1e-6, 0)
    cfg = M.MultiscaleConfig()
    taus = CMP.tau_plan(n // b, n, cfg)
    ok = [CMP.BucketSet(n, b, np.ones(b, complex), CMP.PermutationParams(1, 1, t)) for t in taus]
    with pytest.raises(M.InvalidArgument, match="locate_frequency: round 0 must have tau = 0"):
        CMP.locate_frequency(0, ok[1:], cfg, win)
    with pytest.raises(M.InvalidArgument, match="not enough rounds for the schedule"):
        CMP.locate_frequency(0, ok[:-1], cfg, win)
    with pytest.raises(M.InvalidArgument, match="MultiscaleConfig: l must be >= 2"):
        CMP.locate_frequency(0, ok, M.MultiscaleConfig(1, 1.0), win)
    with pytest.raises(M.InvalidArgument, match="bucket out of range"):
        CMP.locate_frequency(b, ok, cfg, win)
    tiny = [CMP.BucketSet(n, b, np.full(b, 1e300 + 0j) if i else np.full(b, 1e-300 + 0j),
                          CMP.PermutationParams(1, 1, t)) for i, t in enumerate(taus)]
    with pytest.raises(M.DomainError, match="phase_of: zero value"):
        CMP.locate_frequency(0, tiny, cfg, win)


def test_estimate_value_matches_reference(oracle):
    n, b, delta = 1 << 16, 256, 1e-8
    win = CMP.flat_window(n, b, delta)
    rng = np.random.default_rng(4)
    u = rng.integers(0, n, 200)
    y0 = rng.standard_normal(200) + 1j * rng.standard_normal(200)
    got, ok = CMP.estimate_values(y0, u, win)
    assert ok.all()
    ref = np.array([oracle.estimate_value(n, b, delta, y, int(uu)) for y, uu in zip(y0, u)])
    assert np.max(np.abs(got - ref) / np.abs(ref)) <= 1e-13
    assert CMP.estimate_value(y0[0], int(u[0]), win) == got[0]


def sfft4_from_components(x, k, cfg, seed, delta):
    """sfft4 (sfft4.cpp:131-187) over components.run_iteration."""
    n = x.shape[-1]
    iter_cap = int(math.ceil(math.log2(k))) + 2 if k > 1 else 2
    state = CMP.IterationState(k_m=k, b_m=M.Plan(n, k, cfg, delta, "complex128").stats().b_first,
                               delta=delta)
    rng = CMP.Rng(seed)
    stages = []
    for _ in range(iter_cap):
        if state.k_m < 1:
            break
        CMP.run_iteration(x, state, cfg, rng)
        stages.append(state.stages_m)
    acc = state.accumulated
    fs = sorted(acc)
    keep = sorted(sorted(range(len(fs)), key=lambda i: -abs(acc[fs[i]]))[:k])
    return (np.array([fs[i] for i in keep], np.int64),
            np.array([acc[fs[i]] for i in keep], np.complex128), stages, state.samples_round_sum)


@pytest.mark.parametrize("n,k,snr,seed", [(1 << 14, 20, None, 3), (1 << 16, 50, 20.0, 7)])
def test_components_compose_to_sfft4(oracle, n, k, snr, seed):
    """The component API is complete: sfft4 rebuilt from it in the
    reference's order gives exactly the fused GPU transform's output, and
    matches the reference within the north_star tolerance."""
    x = make_signal(oracle, dict(gen="np", n=n, k=k, seed=seed, snr=snr))
    delta = 1e-8 if snr is None else 1e-6
    cfg = M.MultiscaleConfig()
    f, c, stages, round_sum = sfft4_from_components(x, k, cfg, 1000 + seed, delta)
    r = M.sfft4(x, k, cfg, 1000 + seed, delta)
    assert stages == r.stats.stage_counts and round_sum == r.stats.samples_round_sum
    assert np.array_equal(f, r.spectrum.positions)
    assert np.array_equal(c, r.spectrum.coeffs)
    ref = oracle.sfft4(x, k, 16, 1.0, 1000 + seed, delta)
    assert_parity(ref.f, ref.c, f, c, k, delta, 1e-9)
