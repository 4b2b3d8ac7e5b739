"""Signal recipes and parity comparisons shared by the tests."""
import numpy as np

from paper_2011_05698_b200 import splitmix64
from paper_2011_05698_b200.workloads import make_signal_np


def make_signal(o, rec):
    """x for a golden recipe (see tests/golden/make_golden.py)."""
    n, k = rec["n"], rec["k"]
    if rec["gen"] == "ref":
        x, _, _ = o.generate_test_signal(n, k, splitmix64(rec["seed"] ^ 0x51))
        if rec.get("snr") is not None:
            x = o.add_awgn(x, rec["snr"], splitmix64(rec["seed"] ^ 0x52))
    elif rec["gen"] == "np":
        x, _, _ = make_signal_np(n, k, rec["seed"], rec.get("snr"), rec.get("dtype", "complex128"),
                                 rec.get("magnitude", "unit"), rec.get("min_sep", 0))
    elif rec["gen"] == "zero":
        x = np.zeros(n, np.complex128)
    else:
        raise ValueError(rec["gen"])
    if rec.get("dtype") == "complex64":
        x = x.astype(np.complex64)
    return x


def golden_result(rec):
    r = rec["result"]
    f = np.array(r["f"], dtype=np.int64)
    c = np.array([complex(float.fromhex(a), float.fromhex(b)) for a, b in r["c"]],
                 dtype=np.complex128)
    return f, c, r["stats"]


def parity(ref_f, ref_c, f, c, k, delta, tol):
    """(support identical, max relative coefficient error, #entries on the
    absolute floor).  The floor 10*K*delta*max|c| covers late-iteration
    leakage-level entries."""
    ref_f = np.asarray(ref_f)
    f = np.asarray(f)
    if ref_f.shape != f.shape or not np.array_equal(ref_f, f):
        return False, float("inf"), 0
    if ref_f.size == 0:
        return True, 0.0, 0
    ref_c = np.asarray(ref_c)
    floor = 10.0 * k * delta * float(np.max(np.abs(ref_c)))
    den = np.maximum(np.abs(ref_c), floor)
    rel = np.abs(np.asarray(c) - ref_c) / den
    return True, float(np.max(rel)), int(np.sum(np.abs(ref_c) < floor))


def assert_parity(ref_f, ref_c, f, c, k, delta, tol):
    same, err, nfloor = parity(ref_f, ref_c, f, c, k, delta, tol)
    assert same, f"support differs:\n ref {np.asarray(ref_f)[:16]}\n got {np.asarray(f)[:16]}"
    assert err <= tol, f"max relative coefficient error {err:.3g} > {tol:g} ({nfloor} on floor)"
    return err


def prewarm_windows(o, n, k, delta):
    """Design the oracle's windows of a schedule in parallel threads (the
    reference designs take ~20 s each at N=2^22)."""
    import math
    import threading
    b = o.initial_bucket_count(n, k, delta)
    bs = set()
    for _ in range(int(math.ceil(math.log2(k))) + 2):
        bs.add(b)
        b = b // 2 if b > 32 else b
    ts = [threading.Thread(target=o.window, args=(n, bb, delta, False)) for bb in sorted(bs)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
