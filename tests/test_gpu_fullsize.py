"""Full BASELINE size (C4: 1024 x N=2^22, K=64, complex64): size-independent
properties on the whole batch, plus reference parity on a sample.  GPU."""
import numpy as np
import pytest

import paper_2011_05698_b200 as M
from helpers import assert_parity, prewarm_windows

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
N, K, DELTA, B = 1 << 22, 64, 1e-6, 1024


@pytest.fixture(scope="module")
def batch():
    import torch
    from paper_2011_05698_b200.workloads import algo_seed, make_batch, signal_seed
    seeds = [signal_seed(0x7E57, i) for i in range(B)]
    aseeds = np.array([algo_seed(s) for s in seeds], dtype=np.uint64)
    x, _ = make_batch(N, K, seeds, 25.0, torch.device("cuda", 0), "complex64")
    plan = M.Plan(N, K, M.MultiscaleConfig(), DELTA, "complex64")
    return x, aseeds, plan


def run(plan, x, seeds):
    import torch
    b = x.shape[0]
    out = (torch.empty((b, K), dtype=torch.int64, device=x.device),
           torch.empty((b, K), dtype=torch.complex128, device=x.device),
           torch.empty((b,), dtype=torch.int64, device=x.device))
    plan.execute(x, seeds, out=out)
    return [o.cpu().numpy() for o in out]


def test_deterministic(batch):
    x, s, plan = batch
    a = run(plan, x, s)
    b = run(plan, x, s)
    for u, v in zip(a, b):
        assert np.array_equal(u, v)


def test_exact_doubling(batch):
    """sfft4(2x) = 2 sfft4(x) bit-for-bit: scaling by 2 is exact in every
    stage and leaves every decision unchanged."""
    x, s, plan = batch
    f1, c1, n1 = run(plan, x, s)
    f2, c2, n2 = run(plan, x * 2, s)
    assert np.array_equal(n1, n2) and np.array_equal(f1, f2)
    for i in range(B):
        m = n1[i]
        assert np.array_equal(c2[i, :m], 2 * c1[i, :m])


def test_signal_order_invariance(batch):
    x, s, plan = batch
    perm = np.random.default_rng(5).permutation(B)
    import torch
    f1, c1, n1 = run(plan, x, s)
    xp = torch.empty_like(x)
    for i, p in enumerate(perm):  # row copies (torch's gather asserts on 32 GiB)
        xp[i].copy_(x[int(p)])
    f2, c2, n2 = run(plan, xp, s[perm])
    del xp
    assert np.array_equal(f2, f1[perm]) and np.array_equal(c2, c1[perm])


def test_support_sizes(batch):
    x, s, plan = batch
    f, c, n = run(plan, x, s)
    assert np.all(n == K)
    for i in range(B):
        assert np.all(np.diff(f[i]) > 0) and f[i, 0] >= 0 and f[i, -1] < N


def test_reference_sample(batch, oracle):
    """8 signals of the batch through the reference's own sfft4."""
    x, s, plan = batch
    f, c, n = run(plan, x, s)
    prewarm_windows(oracle, N, K, DELTA)
    xs = x[:8].cpu().numpy().astype(np.complex128)
    for i in range(8):
        r = oracle.sfft4(xs[i], K, 16, 1.0, int(s[i]), DELTA)
        assert_parity(r.f, r.c, f[i, :n[i]], c[i, :n[i]], K, DELTA, 1e-4)
