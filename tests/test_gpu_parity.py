"""Parity of the CUDA path (through the C ABI) with the reference.

Bars (BASELINE.json north_star): identical support; per-coefficient relative
error <= 1e-9 for complex128 and <= 1e-4 for complex64 inputs, with the
absolute floor 10*K*delta*max|c| for leakage-level entries.
In practice the encode is bit-identical and coefficients agree to ~1e-15.
Run on a B200: pytest -m gpu.
"""
import hashlib

import numpy as np
import pytest

import paper_2011_05698_b200 as M
from helpers import assert_parity, golden_result, make_signal

pytestmark = pytest.mark.gpu
TOL = {"complex128": 1e-9, "complex64": 1e-4}


def test_device_present():
    assert M.device_count() >= 1


def test_windows_bit_exact(golden):
    g = golden("windows")
    for rec in g["ok"]:
        w, taps = M.window(rec["n"], rec["b"], rec["delta"])
        assert w == rec["w"], (rec["n"], rec["b"], rec["delta"])
        assert hashlib.sha256(taps.astype("<f8").tobytes()).hexdigest() == rec["taps_sha256"]


def test_window_errors_same_messages(golden):
    for rec in golden("windows")["error"]:
        with pytest.raises(M.InvalidArgument) as ei:
            M.window(rec["n"], rec["b"], rec["delta"])
        assert str(ei.value) == rec["msg"]


def test_response_table(golden):
    """G_d from the device table vs response_at: only libm-vs-CUDA cos ulps."""
    for rec in golden("windows")["ok"]:
        offs = [a for a, _ in rec["response"]]
        want = np.array([float.fromhex(h) for _, h in rec["response"]])
        got = M.window_response(rec["n"], rec["b"], rec["delta"], offs)
        assert np.max(np.abs(got - want)) <= 1e-14, (rec["n"], rec["b"])


def test_sfft4_small_goldens(oracle, golden):
    for rec in golden("sfft4_small"):
        x = make_signal(oracle, rec)
        cfg = M.MultiscaleConfig(rec["l"], rec["q"])
        if "error" in rec:
            with pytest.raises(M.InvalidArgument) as ei:
                M.sfft4(x, rec["k"], cfg, rec["algo_seed"], rec["delta"])
            assert str(ei.value) == rec["error"]["msg"]
            continue
        r = M.sfft4(x, rec["k"], cfg, rec["algo_seed"], rec["delta"])
        f, c, stats = golden_result(rec)
        assert_parity(f, c, r.spectrum.positions, r.spectrum.coeffs, rec["k"], rec["delta"],
                      TOL[rec["dtype"]])
        assert r.stats.samples_used == stats["samples_used"]
        assert r.stats.samples_round_sum == stats["samples_round_sum"]
        assert r.stats.iterations == stats["iterations"]
        assert r.stats.b_first == stats["b_first"]
        assert r.stats.stage_counts == stats["stage_counts"]
        assert r.stats.sample_fraction == stats["sample_fraction"]


TRACE_CASES = [
    dict(gen="ref", n=1 << 16, k=50, seed=1, snr=None, l=16, q=1.0, dtype="complex128"),
    dict(gen="ref", n=1 << 20, k=100, seed=2, snr=20.0, l=8, q=2.0, dtype="complex128"),
    dict(gen="np", n=1 << 18, k=64, seed=3, snr=25.0, l=16, q=1.0, dtype="complex64"),
    dict(gen="np", n=1 << 20, k=100, seed=4, snr=20.0, l=4, q=1.0, dtype="complex128"),
]


@pytest.mark.parametrize("rec", TRACE_CASES, ids=lambda r: f"{r['n']}-{r['k']}-{r['l']}-{r['q']}")
def test_stage_parity(oracle, rec):
    """Kernel-level parity against the reference's per-stage trace:
    K1+K2 (encode) bit-identical; K3 (subtract) to rounding; K4 (selection
    order) and K5/K6 (located f per rank) identical; values to rounding."""
    from paper_2011_05698_b200 import splitmix64
    x = make_signal(oracle, rec)
    delta = 1e-6 if rec["snr"] is not None else 1e-8
    a = splitmix64(rec["seed"] ^ 0x53)
    tr = oracle.sfft4_trace(x.astype(np.complex128), rec["k"], rec["l"], rec["q"], a, delta)
    plan = tr["plan"]
    vps = sum(r * b for r, b in zip(plan.rounds, plan.b))
    nsel = sum(plan.budget)
    g = M.trace(x, rec["k"], M.MultiscaleConfig(rec["l"], rec["q"]), a, delta, vps, nsel)
    assert np.array_equal(g["pre"].view(np.float64), tr["pre"].view(np.float64)), "encode"
    scale = np.max(np.abs(tr["pre"]))
    assert np.max(np.abs(g["post"] - tr["post"])) <= 1e-13 * scale, "subtract"
    assert np.array_equal(g["sel_bucket"], tr["sel_bucket"]), "selection order"
    want_f = np.where(tr["sel_status"] == 0, tr["sel_f"], -1)
    assert np.array_equal(g["sel_f"], want_f), "located frequencies"
    ok = want_f >= 0
    assert np.max(np.abs(g["sel_value"][ok] - tr["sel_value"][ok]) /
                  np.abs(tr["sel_value"][ok])) <= 1e-12
    assert_parity(tr["result"].f, tr["result"].c, g["f"], g["c"], rec["k"], delta,
                  TOL[rec["dtype"]])


def test_batch_plan_equals_single_calls(oracle):
    """Plan.execute over a batch == one sfft4 per signal, bitwise, for host
    and device inputs and outputs."""
    import torch
    n, k, delta = 1 << 18, 40, 1e-6
    xs = np.stack([make_signal(oracle, dict(gen="np", n=n, k=k, seed=s, snr=20.0,
                                            dtype="complex64")) for s in range(6)])
    seeds = np.arange(100, 106, dtype=np.uint64)
    plan = M.Plan(n, k, M.MultiscaleConfig(), delta, "complex64")
    f, c, cnt, _ = plan.execute(xs, seeds)
    xd = torch.as_tensor(xs).cuda()
    out = (torch.empty((6, k), dtype=torch.int64, device="cuda"),
           torch.empty((6, k), dtype=torch.complex128, device="cuda"),
           torch.empty((6,), dtype=torch.int64, device="cuda"))
    plan.execute(xd, seeds, out=out)
    for i in range(6):
        r = M.sfft4(xs[i], k, M.MultiscaleConfig(), int(seeds[i]), delta)
        m = int(cnt[i])
        assert np.array_equal(f[i, :m], r.spectrum.positions)
        assert np.array_equal(c[i, :m], r.spectrum.coeffs)
        assert np.array_equal(out[0][i, :m].cpu().numpy(), r.spectrum.positions)
        assert np.array_equal(out[1][i, :m].cpu().numpy(), r.spectrum.coeffs)
        ref = oracle.sfft4(xs[i].astype(np.complex128), k, 16, 1.0, int(seeds[i]), delta)
        assert_parity(ref.f, ref.c, f[i, :m], c[i, :m], k, delta, 1e-4)


def test_device_input_single(oracle):
    import torch
    rec = dict(gen="ref", n=1 << 16, k=50, seed=3, snr=None)
    x = make_signal(oracle, rec)
    from paper_2011_05698_b200 import splitmix64
    a = splitmix64(3 ^ 0x53)
    r_host = M.sfft4(x, 50, seed=a, delta=1e-8)
    r_dev = M.sfft4(torch.as_tensor(x).cuda(), 50, seed=a, delta=1e-8)
    assert np.array_equal(r_host.spectrum.positions, r_dev.spectrum.positions)
    assert np.array_equal(r_host.spectrum.coeffs, r_dev.spectrum.coeffs)


def test_non_finite_input_rejected():
    import torch
    x = np.zeros(1 << 12, np.complex128)
    x[77] = np.nan
    for arg in (x, torch.as_tensor(x).cuda()):
        with pytest.raises(M.InvalidArgument, match="ComplexSignal: non-finite sample"):
            M.sfft4(arg, 10)
    # x is validated before K (proj/src/sfft4.cpp:133-135)
    with pytest.raises(M.InvalidArgument, match="ComplexSignal: non-finite sample"):
        M.sfft4(x, 100000)


def test_bad_length_rejected():
    with pytest.raises(M.InvalidArgument, match="ComplexSignal: n must be a power of two >= 4"):
        M.sfft4(np.zeros(1000, np.complex128), 10)


@pytest.mark.slow
def test_c4_goldens(oracle, golden):
    """Full-size C4 signals (N=2^22, K=64, complex64, 25 dB) vs the reference."""
    for rec in golden("sfft4_c4"):
        x = make_signal(oracle, rec)
        r = M.sfft4(x, rec["k"], M.MultiscaleConfig(), rec["algo_seed"], rec["delta"])
        f, c, stats = golden_result(rec)
        assert_parity(f, c, r.spectrum.positions, r.spectrum.coeffs, rec["k"], rec["delta"], 1e-4)
        assert r.stats.samples_used == stats["samples_used"]


@pytest.mark.slow
def test_c3_goldens(oracle, golden):
    """C3: N=2^24, K=1000, min-separated support, 30 dB, c128 and c64."""
    for rec in golden("sfft4_c3"):
        x = make_signal(oracle, rec)
        r = M.sfft4(x, rec["k"], M.MultiscaleConfig(), rec["algo_seed"], rec["delta"])
        f, c, stats = golden_result(rec)
        assert_parity(f, c, r.spectrum.positions, r.spectrum.coeffs, rec["k"], rec["delta"],
                      TOL[rec["dtype"]])
        assert r.stats.samples_used == stats["samples_used"]


@pytest.mark.slow
def test_large_size_goldens(oracle, golden):
    """C5-law signals that drive the decode's large-size paths (radix-sorted
    selection order at b = 8192, sorted found-map merge at budget 2000,
    sorted K-prune over ~4000 accumulated tones) against the reference."""
    for rec in golden("sfft4_big"):
        x = make_signal(oracle, rec)
        r = M.sfft4(x, rec["k"], M.MultiscaleConfig(), rec["algo_seed"], rec["delta"])
        f, c, stats = golden_result(rec)
        assert_parity(f, c, r.spectrum.positions, r.spectrum.coeffs, rec["k"], rec["delta"],
                      TOL[rec["dtype"]])
        assert r.stats.samples_used == stats["samples_used"]
        assert r.stats.stage_counts == stats["stage_counts"]


@pytest.mark.parametrize("dtype", ["complex64", "complex128"])
def test_sparse_ingest_matches_device_and_dense(oracle, monkeypatch, dtype):
    """Host inputs go through sparse ingest (host gather of the samples the
    transform reads, compact H2D, coalesced encode reads): bitwise equal to
    device-resident inputs and to the dense whole-signal H2D path, across
    several pipeline chunks."""
    import torch
    n, k, delta = 1 << 20, 30, 1e-6
    xs = np.stack([make_signal(oracle, dict(gen="np", n=n, k=k, seed=40 + s, snr=20.0,
                                            dtype=dtype)) for s in range(5)]).astype(dtype)
    seeds = np.arange(500, 505, dtype=np.uint64)
    monkeypatch.setenv("MSFFT_INGEST_CHUNK", "2")
    plan = M.Plan(n, k, M.MultiscaleConfig(), delta, dtype)
    assert 0 < plan.ingest_samples_per_signal <= n // 4
    f, c, cnt, _ = plan.execute(xs, seeds)
    out = (torch.empty((5, k), dtype=torch.int64, device="cuda"),
           torch.empty((5, k), dtype=torch.complex128, device="cuda"),
           torch.empty((5,), dtype=torch.int64, device="cuda"))
    plan.execute(torch.as_tensor(xs).cuda(), seeds, out=out)
    assert np.array_equal(cnt, out[2].cpu().numpy())
    assert np.array_equal(f, out[0].cpu().numpy())
    assert np.array_equal(c, out[1].cpu().numpy())
    monkeypatch.setenv("MSFFT_SPARSE_INGEST", "0")
    dense = M.Plan(n, k, M.MultiscaleConfig(), delta, dtype)
    assert dense.ingest_samples_per_signal == 0
    f2, c2, cnt2, _ = dense.execute(xs, seeds)
    assert np.array_equal(cnt, cnt2) and np.array_equal(f, f2) and np.array_equal(c, c2)
    for i in range(5):
        ref = oracle.sfft4(xs[i].astype(np.complex128), k, 16, 1.0, int(seeds[i]), delta)
        m = int(cnt[i])
        assert_parity(ref.f, ref.c, f[i, :m], c[i, :m], k, delta, TOL[dtype])


def test_sparse_ingest_validates_every_sample():
    """The host scan covers all n samples, not only the gathered ones
    (ComplexSignal::validate, proj/src/signal.cpp:18-26)."""
    n, k = 1 << 20, 10
    plan = M.Plan(n, k, M.MultiscaleConfig(), 1e-6, "complex64")
    assert plan.ingest_samples_per_signal > 0
    x = np.zeros((3, n), np.complex64)
    x[2, n - 1] = np.inf
    with pytest.raises(M.InvalidArgument, match="ComplexSignal: non-finite sample"):
        plan.execute(x, [1, 2, 3])
    x[2, n - 1] = 0
    x[1, 12345] = complex(0, np.nan)
    with pytest.raises(M.InvalidArgument, match="ComplexSignal: non-finite sample"):
        plan.execute(x, [1, 2, 3])
    x[1, 12345] = 0
    f, c, cnt, _ = plan.execute(x, [1, 2, 3])
    assert list(cnt) == [0, 0, 0]


@pytest.mark.parametrize("n,k,dtype,snr", [(1 << 20, 2000, "complex128", 20.0),
                                           (1 << 19, 1200, "complex64", 20.0),
                                           (1 << 18, 3000, "complex128", None),
                                           # budgets >= 4096: K4/K6 orders by radix sort
                                           (1 << 21, 6000, "complex128", 20.0)])
def test_wide_decode_bit_identical_to_cta_decode(oracle, monkeypatch, n, k, dtype, snr):
    """Large single signals decode with the grid-wide kernels (wide_decode.cu);
    outputs must equal the one-CTA decode (decode_body.cuh) bit for bit."""
    x, _, _ = __import__("paper_2011_05698_b200.workloads", fromlist=["x"]).make_signal_np(
        n, k, 5, snr, dtype, "loguniform_0.1_10")
    x = x.astype(dtype)
    delta = 1e-6 if snr is not None else 1e-8
    res = []
    for wide in ("8", "0"):
        monkeypatch.setenv("MSFFT_WIDE_MAX_BATCH", wide)
        plan = M.Plan(n, k, M.MultiscaleConfig(), delta, dtype)
        res.append(plan.execute(x[None, :], [123]))
    (f1, c1, n1, _), (f0, c0, n0, _) = res
    assert int(n1[0]) == int(n0[0]) > 0
    assert np.array_equal(f1, f0) and np.array_equal(c1, c0)


@pytest.mark.parametrize("l,q", [(4, 1.0), (4, 2.0), (8, 2.0), (32, 1.0)])
def test_wide_decode_other_multiscale_configs(oracle, monkeypatch, l, q):
    """The wide decode's locate kernel with other lane-group sizes (l = 4, 8,
    32 -> groups of 4, 8, 32 lanes) and stage counts: (4, 2) has more stages
    than the shared staging of k5_locate holds for 64 groups per CTA, so it
    takes the separate k5_stage_phase launch; the others compute their stage
    phases inside k5_locate.  Each equals the one-CTA decode bit for bit."""
    n, k = 1 << 20, 1500
    x, _, _ = __import__("paper_2011_05698_b200.workloads", fromlist=["x"]).make_signal_np(
        n, k, 21, 25.0, "complex128", "loguniform_0.1_10")
    res = []
    for wide in ("8", "0"):
        monkeypatch.setenv("MSFFT_WIDE_MAX_BATCH", wide)
        plan = M.Plan(n, k, M.MultiscaleConfig(l, q), 1e-6, "complex128")
        res.append(plan.execute(x[None, :], [4242]))
    (f1, c1, n1, _), (f0, c0, n0, _) = res
    assert int(n1[0]) == int(n0[0]) > 0
    assert np.array_equal(f1, f0) and np.array_equal(c1, c0)


@pytest.mark.parametrize("knob,values", [("MSFFT_ENC_SPLIT", ("1", "0")),
                                         ("MSFFT_WIDE_PDL", ("1", "0")),
                                         ("MSFFT_WIDE_GRAPH", ("1", "0")),
                                         ("MSFFT_WIDE_GROUPS", ("5", "1", "3")),
                                         ("MSFFT_FFT_TWO_PASS", ("1", "0"))])
def test_launch_knobs_bit_identical(oracle, monkeypatch, knob, values):
    """Launch-shape knobs change only how the work is spread over CTAs and
    launches: per-segment encode tasks (small launches), programmatic edges
    and the CUDA graph of the wide decode, the wide decode overlapped with
    the encode in iteration groups.  Results are bit-identical."""
    monkeypatch.setenv("MSFFT_WIDE_OVERLAP_MIN", "0")
    n, k = 1 << 19, 1200
    x, _, _ = __import__("paper_2011_05698_b200.workloads", fromlist=["x"]).make_signal_np(
        n, k, 9, 20.0, "complex128", "loguniform_0.1_10")
    res = []
    for v in values:
        monkeypatch.setenv(knob, v)
        plan = M.Plan(n, k, M.MultiscaleConfig(), 1e-6, "complex128")
        res.append(plan.execute(x[None, :], [321]))
        res.append(plan.execute(x[None, :], [321], assume_valid=True))  # graph replay
    f0, c0, n0, _ = res[0]
    assert int(n0[0]) > 0
    for f, c, cnt, _ in res[1:]:
        assert int(cnt[0]) == int(n0[0])
        assert np.array_equal(f, f0) and np.array_equal(c, c0)


def test_sparse_ingest_split_validation(oracle, monkeypatch):
    """Pinned host batches split validation between the copy engine + device
    check (first rows) and the host's fused scan+gather (the rest): a
    non-finite sample anywhere in any row raises, and clean results equal the
    device-resident path bit for bit."""
    import torch
    n, k = 1 << 20, 20
    monkeypatch.setenv("MSFFT_DMA_VALIDATE_SHARE", "0.5")
    monkeypatch.setenv("MSFFT_INGEST_CHUNK", "3")
    plan = M.Plan(n, k, M.MultiscaleConfig(), 1e-6, "complex64")
    assert plan.ingest_samples_per_signal > 0
    xs = np.stack([make_signal(oracle, dict(gen="np", n=n, k=k, seed=70 + s, snr=20.0,
                                            dtype="complex64")) for s in range(8)])
    xh = torch.from_numpy(xs).pin_memory()
    seeds = np.arange(900, 908, dtype=np.uint64)
    f, c, cnt, _ = plan.execute(xh, seeds)
    out = (torch.empty((8, k), dtype=torch.int64, device="cuda"),
           torch.empty((8, k), dtype=torch.complex128, device="cuda"),
           torch.empty((8,), dtype=torch.int64, device="cuda"))
    plan.execute(xh.cuda(), seeds, out=out)
    assert np.array_equal(f, out[0].cpu().numpy()) and np.array_equal(c, out[1].cpu().numpy())
    for row, col in ((1, 5), (6, n - 1), (7, 0), (4, n // 2 + 3)):
        xb = xh.clone()
        xb[row, col] = complex(float("nan"), 0.0)
        with pytest.raises(M.InvalidArgument, match="ComplexSignal: non-finite sample"):
            plan.execute(xb.pin_memory(), seeds)


@pytest.mark.parametrize("n,k,kind", [
    (64, 8, "max_k"),            # K = n/8, the largest K sfft4 accepts (sfft4.cpp:135)
    (1 << 12, 512, "max_k"),
    (8, 1, "tiny"),              # smallest n with K >= 1
    (16, 2, "tiny"),
    (1 << 12, 16, "equal"),      # equal magnitudes: stable tie-breaks in selection / K-prune
    (1 << 14, 40, "range"),      # magnitudes over 12 decades
])
def test_edge_cases_match_reference(oracle, n, k, kind):
    rng = np.random.default_rng(n + k)
    if kind == "equal":
        f = np.sort(rng.choice(n, k, replace=False))
        c = np.full(k, 1.0 + 0.0j)
        x = np.zeros(n, np.complex128)
        x[f] = c
        x = np.fft.ifft(x) * n
    elif kind == "range":
        f = np.sort(rng.choice(n, k, replace=False))
        c = 10.0 ** rng.uniform(-6, 6, k) * np.exp(2j * np.pi * rng.random(k))
        spec = np.zeros(n, np.complex128)
        spec[f] = c
        x = np.fft.ifft(spec) * n
    else:
        x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    for delta in (1e-8, 1e-6):
        try:
            ref = oracle.sfft4(x, k, 16, 1.0, 77, delta)
        except Exception as e:  # noqa: BLE001  the GPU must raise the same error
            with pytest.raises((M.InvalidArgument, M.DomainError)) as ours:
                M.sfft4(x, k, M.MultiscaleConfig(), 77, delta)
            assert str(ours.value) == str(e)
            continue
        r = M.sfft4(x, k, M.MultiscaleConfig(), 77, delta)
        assert_parity(ref.f, ref.c, r.spectrum.positions, r.spectrum.coeffs, k, delta, 1e-9)


def test_async_execute(oracle):
    """MSFFT_FLAG_ASYNC: enqueue-only calls give the synchronous results,
    the σ plan is reused only while the seeds repeat, decode/validation
    errors are raised by sync() and then cleared, host inputs are refused."""
    import torch
    n, k = 1 << 18, 40
    xs = np.stack([make_signal(oracle, dict(gen="np", n=n, k=k, seed=s, snr=20.0,
                                            dtype="complex64")) for s in range(4)])
    plan = M.Plan(n, k, M.MultiscaleConfig(), 1e-6, "complex64")
    xd = torch.as_tensor(xs).cuda()
    outs = []
    for seeds in (np.arange(10, 14, dtype=np.uint64), np.arange(10, 14, dtype=np.uint64),
                  np.arange(20, 24, dtype=np.uint64)):
        o = (torch.empty((4, k), dtype=torch.int64, device="cuda"),
             torch.empty((4, k), dtype=torch.complex128, device="cuda"),
             torch.empty((4,), dtype=torch.int64, device="cuda"))
        plan.execute(xd, seeds, out=o, async_=True)
        outs.append((seeds, o))
    plan.sync()
    for seeds, o in outs:
        f, c, cnt, _ = plan.execute(xs, seeds)
        assert np.array_equal(cnt, o[2].cpu().numpy())
        assert np.array_equal(f, o[0].cpu().numpy()) and np.array_equal(c, o[1].cpu().numpy())
    assert not np.array_equal(outs[0][1][0].cpu().numpy(), outs[2][1][0].cpu().numpy())
    bad = xd.clone()
    bad[2, 17] = complex(float("nan"), 0)
    plan.execute(bad, outs[0][0], out=outs[0][1], async_=True)
    with pytest.raises(M.InvalidArgument, match="ComplexSignal: non-finite sample"):
        plan.sync()
    plan.execute(xd, outs[0][0], out=outs[0][1], async_=True)
    plan.sync()  # cleared
    with pytest.raises(M.InvalidArgument, match="MSFFT_FLAG_ASYNC needs device input and output"):
        plan.execute(xs, outs[0][0], async_=True)


def test_async_pdl_chain(oracle, monkeypatch):
    """Batches large enough for chained programmatic launches (step i+1 starts
    while step i's last decodes run; opt-in MSFFT_PDL=1): every step's outputs
    equal the synchronous path's, over alternating and changing seed sets."""
    import torch
    monkeypatch.setenv("MSFFT_PDL", "1")
    n, k, B = 1 << 18, 40, 320
    rng = np.random.default_rng(5)
    xs = (rng.standard_normal((B, n)) + 1j * rng.standard_normal((B, n))).astype(np.complex64)
    xs[:, 0] += 50.0  # a strong tone so every signal has support
    plan = M.Plan(n, k, M.MultiscaleConfig(), 1e-6, "complex64")
    xd = torch.as_tensor(xs).cuda()
    seed_sets = [np.arange(1000, 1000 + B, dtype=np.uint64) + np.uint64(7919 * i) for i in range(3)]
    order = [0, 1, 0, 1, 2, 1, 2, 0]
    outs = []
    for i in order:
        o = (torch.empty((B, k), dtype=torch.int64, device="cuda"),
             torch.empty((B, k), dtype=torch.complex128, device="cuda"),
             torch.empty((B,), dtype=torch.int64, device="cuda"))
        plan.execute(xd, seed_sets[i], out=o, assume_valid=True, async_=True)
        outs.append(o)
    plan.sync()
    ref = {}
    for i in set(order):
        o = (torch.empty((B, k), dtype=torch.int64, device="cuda"),
             torch.empty((B, k), dtype=torch.complex128, device="cuda"),
             torch.empty((B,), dtype=torch.int64, device="cuda"))
        plan.execute(xd, seed_sets[i], out=o, assume_valid=True)
        ref[i] = [t.cpu().numpy() for t in o]
    for i, o in zip(order, outs):
        got = [t.cpu().numpy() for t in o]
        assert all(np.array_equal(a, b) for a, b in zip(got, ref[i]))


def test_async_pdl_shared_outputs(monkeypatch):
    """consecutive asynchronous calls that share one output set
    (different seeds) must not chain programmatically -- a late decode of
    call i would overwrite call i+1's result.  The final outputs equal the
    last call's synchronous result."""
    import torch
    monkeypatch.setenv("MSFFT_PDL", "1")
    n, k, B = 1 << 18, 40, 320
    rng = np.random.default_rng(6)
    xs = (rng.standard_normal((B, n)) + 1j * rng.standard_normal((B, n))).astype(np.complex64)
    xs[:, 3] += 50.0
    plan = M.Plan(n, k, M.MultiscaleConfig(), 1e-6, "complex64")
    xd = torch.as_tensor(xs).cuda()
    o = (torch.empty((B, k), dtype=torch.int64, device="cuda"),
         torch.empty((B, k), dtype=torch.complex128, device="cuda"),
         torch.empty((B,), dtype=torch.int64, device="cuda"))
    seeds = [np.arange(B, dtype=np.uint64) * np.uint64(31) + np.uint64(i) for i in range(6)]
    for sd in seeds:
        plan.execute(xd, sd, out=o, assume_valid=True, async_=True)
    plan.sync()
    got = [t.cpu().numpy() for t in o]
    ref = plan.execute(xs, seeds[-1], assume_valid=True)[:3]
    assert all(np.array_equal(a, b) for a, b in zip(got, ref))


@pytest.mark.slow
def test_c3_more_seeds(oracle, golden):
    """C3 on two more seeds (302, 303), complex128 and complex64."""
    for rec in golden("sfft4_c3_more"):
        x = make_signal(oracle, rec)
        r = M.sfft4(x, rec["k"], M.MultiscaleConfig(), rec["algo_seed"], rec["delta"])
        f, c, stats = golden_result(rec)
        assert_parity(f, c, r.spectrum.positions, r.spectrum.coeffs, rec["k"], rec["delta"],
                      TOL[rec["dtype"]])
        assert r.stats.samples_used == stats["samples_used"]
        assert r.stats.samples_round_sum == stats["samples_round_sum"]
        assert r.stats.stage_counts == stats["stage_counts"]


@pytest.mark.slow
def test_c5_full_size_golden(oracle, golden):
    """C5 at full size (BASELINE.json configs[4]: N=2^27, K=10^4, c128,
    log-uniform |c| in [0.1, 10], 20 dB) against the reference's own sfft4
    run on the same bytes (tests/golden/make_golden.py c5, ~1-2 h of CPU):
    the 12 windows bit-exact (w and sha256 of the taps, window.cpp:105-177),
    identical support, coefficients within 1e-9 (with the 10*K*delta floor),
    identical stats -- through the fused one-shot path and through the
    tap-range sharded split (8 parts summed, then decoded)."""
    import hashlib
    import torch
    rec = golden("sfft4_c5")
    for wrec in rec["windows"]:
        w, taps = M.window(wrec["n"], wrec["b"], wrec["delta"])
        assert w == wrec["w"], wrec["b"]
        assert hashlib.sha256(taps.astype("<f8").tobytes()).hexdigest() == wrec["taps_sha256"]
    x = make_signal(oracle, rec)
    f, c, stats = golden_result(rec)
    k, delta = rec["k"], rec["delta"]
    plan = M.Plan(rec["n"], k, M.MultiscaleConfig(rec["l"], rec["q"]), delta, "complex128")
    xd = torch.as_tensor(x).cuda().reshape(1, -1)
    del x
    seeds = np.array([rec["algo_seed"]], np.uint64)
    out = (torch.empty((1, k), dtype=torch.int64, device="cuda"),
           torch.empty((1, k), dtype=torch.complex128, device="cuda"),
           torch.empty((1,), dtype=torch.int64, device="cuda"))
    plan.execute(xd, seeds, out=out)
    m = int(out[2].item())
    err = assert_parity(f, c, out[0][0, :m].cpu().numpy(), out[1][0, :m].cpu().numpy(), k, delta,
                        1e-9)
    st = plan.stats()
    assert st.samples_round_sum == stats["samples_round_sum"]
    assert st.b_first == stats["b_first"] and st.iterations == stats["iterations"]
    assert st.stage_counts == stats["stage_counts"]
    r1 = M.sfft4(xd[0], k, M.MultiscaleConfig(rec["l"], rec["q"]), rec["algo_seed"], delta)
    assert r1.stats.samples_used == stats["samples_used"]
    # tap-range sharded over 8 parts (what 8 ranks + one all-reduce compute)
    y = None
    for p in range(8):
        part = plan.encode_values_part(xd, seeds, p, 8)
        y = part if y is None else y + part
    fs, cs, ns = plan.decode_values(y, seeds, folds=True)
    ms = int(ns[0].item())
    err8 = assert_parity(f, c, fs[0, :ms].cpu().numpy(), cs[0, :ms].cpu().numpy(), k, delta, 1e-9)
    print(f"C5 parity: {m} entries, max rel err {err:.3g} (one GPU), {err8:.3g} (8 parts)")


def test_wide_decode_clustered_spectrum(monkeypatch):
    """a support packed into a narrow band puts every accepted
    candidate of an iteration into one or a few buckets of the K6 (f, rank)
    bucket sort (budgets >= 2048); the wide decode must still equal the
    one-CTA decode bit for bit (and finish in normal time)."""
    n, k = 1 << 21, 3000
    rng = np.random.default_rng(11)
    f0 = 123457
    pos = np.sort(f0 + rng.choice(4096, k, replace=False)).astype(np.int64)
    spec = np.zeros(n, np.complex128)
    spec[pos] = 10.0 ** rng.uniform(-1, 1, k) * np.exp(2j * np.pi * rng.random(k))
    x = np.fft.ifft(spec) * n
    noise = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    x = x + np.sqrt(np.sum(np.abs(x) ** 2) * 1e-2 / np.sum(np.abs(noise) ** 2)) * noise
    res = []
    for wide in ("8", "0"):
        monkeypatch.setenv("MSFFT_WIDE_MAX_BATCH", wide)
        plan = M.Plan(n, k, M.MultiscaleConfig(), 1e-6, "complex128")
        res.append(plan.execute(x[None, :], [77]))
    (f1, c1, n1, _), (f0_, c0, n0, _) = res
    assert int(n1[0]) == int(n0[0]) > 0
    assert np.array_equal(f1, f0_) and np.array_equal(c1, c0)


def test_concurrent_one_shot_calls(oracle):
    """The reference's run_sweep calls sfft4 from several threads at once
    (bench.cpp:242-280).  Same-geometry one-shot calls from 4 threads lease
    separate plans (up to 4 per geometry) and return exactly the sequential
    results."""
    import concurrent.futures as cf
    n, k = 1 << 16, 50
    xs = [oracle.generate_test_signal(n, k, M.splitmix64(s ^ 0x51))[0] for s in range(8)]
    seeds = [M.splitmix64(s ^ 0x53) for s in range(8)]
    seq = [M.sfft4(x, k, M.MultiscaleConfig(), sd, 1e-8) for x, sd in zip(xs, seeds)]
    with cf.ThreadPoolExecutor(4) as ex:
        par = list(ex.map(lambda a: M.sfft4(a[0], k, M.MultiscaleConfig(), a[1], 1e-8),
                          zip(xs, seeds)))
    for a, b in zip(seq, par):
        assert np.array_equal(a.spectrum.positions, b.spectrum.positions)
        assert np.array_equal(a.spectrum.coeffs, b.spectrum.coeffs)


@pytest.mark.parametrize("batch,n,k,l,q", [(1, 1 << 18, 64, 16, 1.0), (5, 1 << 18, 64, 16, 1.0),
                                           (16, 1 << 18, 64, 16, 1.0),
                                           # b = 512, 256, ...: the gated bucket FFT in between
                                           (1, 1 << 20, 100, 4, 1.0), (3, 1 << 20, 100, 8, 2.0)])
def test_gated_decode_matches_fused_and_serial(oracle, monkeypatch, batch, n, k, l, q):
    import torch
    """Small batches run the encode and a gated decode launch behind it (the
    decode starts while the encode runs and waits per iteration on the
    encode's (or, b > 256, the gated bucket FFT's) completion counters).
    Results equal the ungated launches (the fused persistent kernel, or
    encode -> FFT -> decode when b > 256) and the serial path bit for bit, on repeated calls (the
    last decode CTA resets the counters) and after a call whose input fails
    validation (its decodes are skipped; the counters must still drain) --
    with host and device-resident inputs (the latter through the device
    compact gather and, on repeated buffers, a replayed CUDA graph)."""
    mk = __import__("paper_2011_05698_b200.workloads", fromlist=["x"]).make_signal_np
    x = np.stack([mk(n, k, 40 + i, 25.0, "complex64")[0] for i in range(batch)]).astype(np.complex64)
    seeds = [1000 + i for i in range(batch)]
    res = {}
    for name, gmax, graph in (("ungated", "0", "1"), ("gated", "64", "1"), ("gated_nograph", "64", "0")):
        monkeypatch.setenv("MSFFT_GATED_MAX_BATCH", gmax)
        monkeypatch.setenv("MSFFT_GATED_GRAPH", graph)
        plan = M.Plan(n, k, M.MultiscaleConfig(l, q), 1e-6, "complex64")
        out = [plan.execute(x, seeds)]
        bad = x.copy()
        bad[batch - 1, 777] = np.nan
        with pytest.raises(M.InvalidArgument, match="non-finite"):
            plan.execute(bad, seeds)
        out.append(plan.execute(x, seeds))
        out.append(plan.execute(x, seeds, assume_valid=True))
        # device-resident input and outputs: the device compact gather and,
        # from the second call on the same buffers, the captured CUDA graph
        xd = torch.as_tensor(x).to("cuda")
        od = (torch.empty((batch, k), dtype=torch.int64, device="cuda"),
              torch.empty((batch, k), dtype=torch.complex128, device="cuda"),
              torch.empty((batch,), dtype=torch.int64, device="cuda"))
        for i in range(4):
            od[0].fill_(-7)
            plan.execute(xd, seeds, out=od, assume_valid=i % 2 == 1)
            out.append(tuple(t.cpu().numpy() for t in od) + (0.0,))
        bad_d = torch.as_tensor(bad).to("cuda")
        with pytest.raises(M.InvalidArgument, match="non-finite"):
            plan.execute(bad_d, seeds, out=od)
        plan.execute(xd, seeds, out=od)
        out.append(tuple(t.cpu().numpy() for t in od) + (0.0,))
        res[name] = out
        if name == "gated":
            res["serial"] = [plan.execute(x, seeds, serial=True)]
    f0, c0, n0, _ = res["ungated"][0]
    assert (n0 > 0).all()
    for name in res:
        for f, c, cnt, _ in res[name]:
            assert np.array_equal(cnt, n0) and np.array_equal(f, f0) and np.array_equal(c, c0), name


def test_wide_overlapped_batch(oracle, monkeypatch):
    """Large signals decoded while their later iterations are still being
    encoded (iteration groups, the wide decode on its own stream): a batch of
    three signals equals the encode-everything-first path and each signal
    transformed alone, bit for bit, with device-resident and host input."""
    import torch
    mk = __import__("paper_2011_05698_b200.workloads", fromlist=["x"]).make_signal_np
    n, k = 1 << 19, 1200
    x = np.stack([mk(n, k, 70 + i, 20.0, "complex128", "loguniform_0.1_10")[0] for i in range(3)])
    seeds = [11, 12, 13]
    res = {}
    monkeypatch.setenv("MSFFT_WIDE_OVERLAP_MIN", "0")  # small enough for a test
    for g in ("5", "1"):
        monkeypatch.setenv("MSFFT_WIDE_GROUPS", g)
        plan = M.Plan(n, k, M.MultiscaleConfig(), 1e-6, "complex128")
        res[g] = plan.execute(x, seeds)
        xd = torch.as_tensor(x).to("cuda")
        od = (torch.empty((3, k), dtype=torch.int64, device="cuda"),
              torch.empty((3, k), dtype=torch.complex128, device="cuda"),
              torch.empty((3,), dtype=torch.int64, device="cuda"))
        for i in range(2):
            plan.execute(xd, seeds, out=od, assume_valid=i == 1)
            f, c, cnt = (t.cpu().numpy() for t in od)
            assert np.array_equal(f, res[g][0]) and np.array_equal(c, res[g][1])
        if g == "5":
            for i in range(3):
                f1, c1, n1, _ = plan.execute(x[i:i + 1], [seeds[i]])
                assert np.array_equal(f1[0], res[g][0][i]) and np.array_equal(c1[0], res[g][1][i])
    assert (res["5"][2] > 0).all()
    assert np.array_equal(res["5"][0], res["1"][0]) and np.array_equal(res["5"][1], res["1"][1])
