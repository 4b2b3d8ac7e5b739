"""Index-range sharding of one signal (SURVEY.md 8(e), C5 law) through the
split-phase C ABI (msfft_encode_values / msfft_decode_values).

On one GPU the G ranks are run one after another (no rank waits on another):
each encodes its slice x[lo_r, hi_r) into a partial bucket vector, the
partials are summed in rank order (what the all-reduce computes), and the
decode runs on the sum.  The result must meet the same parity bar against the
reference as the single-GPU path.  The NCCL/gloo collective itself is covered
by tests/test_dist_gloo.py.
"""
import numpy as np
import pytest

import paper_2011_05698_b200 as M
from paper_2011_05698_b200.dist import index_range
from helpers import assert_parity, golden_result, make_signal

pytestmark = pytest.mark.gpu
TOL = {"complex128": 1e-9, "complex64": 1e-4}


def _sharded(plan, xd, seeds, world):
    import torch
    n = xd.shape[-1]
    y = None
    for r in range(world):
        lo, hi = index_range(n, r, world)
        part = plan.encode_values(xd[:, lo:hi].contiguous(), seeds, lo)
        y = part if y is None else y + part
    f, c, cnt = plan.decode_values(y.contiguous(), seeds)
    torch.cuda.synchronize()
    return f.cpu().numpy(), c.cpu().numpy(), cnt.cpu().numpy()


def _cases(golden):
    return [r for r in golden("sfft4_small") if "result" in r and r["k"] >= 10 and r["n"] >= 1 << 12]


def test_full_range_split_equals_execute(oracle, golden):
    """encode_values over [0, n) + decode_values == execute, bitwise."""
    import torch
    for rec in _cases(golden)[:6]:
        x = make_signal(oracle, rec)
        dt = rec["dtype"]
        plan = M.Plan(rec["n"], rec["k"], M.MultiscaleConfig(rec["l"], rec["q"]), rec["delta"], dt)
        seeds = np.array([rec["algo_seed"]], np.uint64)
        f0, c0, n0, _ = plan.execute(x[None, :], seeds)
        xd = torch.as_tensor(x[None, :]).cuda()
        f1, c1, n1 = _sharded(plan, xd, seeds, 1)
        assert int(n1[0]) == int(n0[0])
        m = int(n0[0])
        assert np.array_equal(f1[0, :m], f0[0, :m])
        assert np.array_equal(c1[0, :m], c0[0, :m])


@pytest.mark.parametrize("world", [2, 3, 8])
def test_sharded_matches_reference(oracle, golden, world):
    import torch
    for rec in _cases(golden):
        x = make_signal(oracle, rec)
        plan = M.Plan(rec["n"], rec["k"], M.MultiscaleConfig(rec["l"], rec["q"]), rec["delta"],
                      rec["dtype"])
        seeds = np.array([rec["algo_seed"]], np.uint64)
        xd = torch.as_tensor(x[None, :]).cuda()
        f, c, cnt = _sharded(plan, xd, seeds, world)
        gf, gc, _ = golden_result(rec)
        m = int(cnt[0])
        assert_parity(gf, gc, f[0, :m], c[0, :m], rec["k"], rec["delta"], TOL[rec["dtype"]])


def test_sharded_batch_and_wide_buckets(oracle, golden):
    """A batch of signals and an iteration with b > 256 (separate bucket FFT):
    the large-size golden at N=2^19 (b1 = 4096) sharded over 4 ranks."""
    import torch
    recs = [r for r in golden("sfft4_big") if r["n"] == 1 << 19]
    for rec in recs:
        x = make_signal(oracle, rec)
        plan = M.Plan(rec["n"], rec["k"], M.MultiscaleConfig(rec["l"], rec["q"]), rec["delta"],
                      rec["dtype"])
        seeds = np.array([rec["algo_seed"]] * 2, np.uint64)
        xd = torch.as_tensor(np.stack([x, x])).cuda()
        f, c, cnt = _sharded(plan, xd, seeds, 4)
        gf, gc, _ = golden_result(rec)
        for i in range(2):
            m = int(cnt[i])
            assert_parity(gf, gc, f[i, :m], c[i, :m], rec["k"], rec["delta"], TOL[rec["dtype"]])


def test_encode_values_rejects_bad_ranges():
    import torch
    plan = M.Plan(1 << 12, 10, M.MultiscaleConfig(), 1e-6, "complex128")
    x = torch.zeros((1, 1 << 11), dtype=torch.complex128, device="cuda")
    with pytest.raises(M.InvalidArgument, match="x_lo < x_hi <= n"):
        plan.encode_values(x, [1], (1 << 11) + 1)
    with pytest.raises(M.InvalidArgument, match="x_lo < x_hi <= n"):
        plan.encode_values(x, [1], -1)
    x[0, 5] = float("nan")
    with pytest.raises(M.InvalidArgument, match="ComplexSignal: non-finite sample"):
        plan.encode_values(x, [1], 0)


def _tap_sharded(plan, xd, seeds, world):
    """Tap-range sharding (x replicated): the parts' partial vectors summed in
    rank order (what the all-reduce computes), then decoded."""
    import torch
    y = None
    for r in range(world):
        part = plan.encode_values_part(xd, seeds, r, world)
        y = part if y is None else y + part
    y_sum = y.clone()
    f, c, cnt = plan.decode_values(y.contiguous(), seeds, folds=True)  # consumes y
    torch.cuda.synchronize()
    return f.cpu().numpy(), c.cpu().numpy(), cnt.cpu().numpy(), y_sum


def test_tap_split_one_part_equals_execute(oracle, golden):
    """encode_values_part(0, 1) + decode_values == execute, bitwise."""
    import torch
    for rec in _cases(golden)[:6]:
        x = make_signal(oracle, rec)
        plan = M.Plan(rec["n"], rec["k"], M.MultiscaleConfig(rec["l"], rec["q"]), rec["delta"],
                      rec["dtype"])
        seeds = np.array([rec["algo_seed"]], np.uint64)
        f0, c0, n0, _ = plan.execute(x[None, :], seeds)
        f1, c1, n1, _ = _tap_sharded(plan, torch.as_tensor(x[None, :]).cuda(), seeds, 1)
        m = int(n0[0])
        assert int(n1[0]) == m
        assert np.array_equal(f1[0, :m], f0[0, :m]) and np.array_equal(c1[0, :m], c0[0, :m])


@pytest.mark.parametrize("world", [2, 3, 8])
def test_tap_sharded_matches_reference(oracle, golden, world):
    import torch
    for rec in _cases(golden):
        x = make_signal(oracle, rec)
        plan = M.Plan(rec["n"], rec["k"], M.MultiscaleConfig(rec["l"], rec["q"]), rec["delta"],
                      rec["dtype"])
        seeds = np.array([rec["algo_seed"]], np.uint64)
        xd = torch.as_tensor(x[None, :]).cuda()
        f, c, cnt, y = _tap_sharded(plan, xd, seeds, world)
        y1 = plan.encode_values_part(xd, seeds, 0, 1)
        # the partial sums add up to the single-part vector up to rounding
        scale = float(torch.max(torch.abs(y1)).item())
        assert float(torch.max(torch.abs(y - y1)).item()) <= 1e-13 * max(scale, 1e-300)
        gf, gc, _ = golden_result(rec)
        m = int(cnt[0])
        assert_parity(gf, gc, f[0, :m], c[0, :m], rec["k"], rec["delta"], TOL[rec["dtype"]])


def test_tap_sharded_large_golden(oracle, golden):
    """The C5-law large-size goldens (b up to 8192, budget 2000) over 4 parts."""
    import torch
    for rec in golden("sfft4_big"):
        x = make_signal(oracle, rec)
        plan = M.Plan(rec["n"], rec["k"], M.MultiscaleConfig(rec["l"], rec["q"]), rec["delta"],
                      rec["dtype"])
        seeds = np.array([rec["algo_seed"]], np.uint64)
        f, c, cnt, _ = _tap_sharded(plan, torch.as_tensor(x[None, :]).cuda(), seeds, 4)
        gf, gc, _ = golden_result(rec)
        m = int(cnt[0])
        assert_parity(gf, gc, f[0, :m], c[0, :m], rec["k"], rec["delta"], TOL[rec["dtype"]])
