"""Ad-hoc GPU diagnostics (not collected by pytest): window, encode and full
sfft4 parity against the compiled reference on a few small cases."""
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/tests/", 1)[0])
import paper_2011_05698_b200 as M  # noqa: E402
from oracle import load  # noqa: E402

o = load("reference")


def sm(x):
    return M.splitmix64(x)


def check_window(n, b, d):
    t = time.time()
    w, g = M.window(n, b, d)
    t1 = time.time() - t
    t = time.time()
    wr, gr = o.window(n, b, d)
    t2 = time.time() - t
    same = w == wr and np.array_equal(g, gr)
    maxd = np.max(np.abs(g - gr)) if w == wr else float("nan")
    L = n // b
    idx = np.arange(-(3 * L // 2 + 1), 3 * L // 2 + 2, max(1, L // 64))
    gm = M.window_response(n, b, d, idx)
    gref = o.response_at(n, b, d, idx)
    rel = np.max(np.abs(gm - gref)) / np.max(np.abs(gref))
    print(f"window n={n} b={b} d={d}: w={w} ref={wr} bitexact={same} maxdiff={maxd:.3g} "
          f"resp_rel={rel:.3g} gpu {t1:.2f}s ref {t2:.2f}s", flush=True)


def check_sfft(n, k, seed, snr=None, l=16, q=1.0, dtype=np.complex128):
    x, f, c = o.generate_test_signal(n, k, sm(seed ^ 0x51))
    delta = 1e-8
    if snr is not None:
        x = o.add_awgn(x, snr, sm(seed ^ 0x52))
        delta = 1e-6
    x = x.astype(dtype)
    a = sm(seed ^ 0x53)
    tr = o.sfft4_trace(x.astype(np.complex128), k, l, q, a, delta)
    plan = tr["plan"]
    vps = sum(r * b for r, b in zip(plan.rounds, plan.b))
    nsel = sum(plan.budget)
    t = time.time()
    g = M.trace(x, k, M.MultiscaleConfig(l, q), a, delta, values_per_signal=vps, selections=nsel)
    dt = time.time() - t
    pre_exact = np.array_equal(g["pre"], tr["pre"])
    pre_rel = np.max(np.abs(g["pre"] - tr["pre"])) / np.max(np.abs(tr["pre"]))
    post_rel = np.max(np.abs(g["post"] - tr["post"])) / np.max(np.abs(tr["post"]))
    rf, rc = tr["result"].f, tr["result"].c
    supp = np.array_equal(g["f"], rf)
    if supp:
        floor = 10 * k * delta * np.max(np.abs(rc))
        err = np.max(np.abs(g["c"] - rc) / np.maximum(np.abs(rc), floor))
    else:
        err = float("nan")
    r = M.sfft4(x, k, M.MultiscaleConfig(l, q), a, delta)
    ref = o.sfft4(x.astype(np.complex128), k, l, q, a, delta)
    same_api = np.array_equal(r.spectrum.positions, ref.f)
    print(f"sfft n={n} k={k} seed={seed} snr={snr} l={l} q={q} {np.dtype(dtype).name}: "
          f"pre_exact={pre_exact} pre_rel={pre_rel:.3g} post_rel={post_rel:.3g} "
          f"support={supp} ({len(g['f'])}/{len(rf)}) coef_rel={err:.3g} api_support={same_api} "
          f"stats_ok={r.stats.samples_used == ref.stats['samples_used'] and r.stats.samples_round_sum == ref.stats['samples_round_sum']} "
          f"trace {dt:.2f}s", flush=True)
    if not supp:
        print("  gpu f", g["f"][:20], "\n  ref f", rf[:20])
        # first diverging selection
        rb, rfs = tr["sel_bucket"], np.where(tr["sel_status"] == 0, tr["sel_f"], -1)
        off = 0
        for m, bud in enumerate(plan.budget):
            gb, gf = g["sel_bucket"][off:off + bud], g["sel_f"][off:off + bud]
            if not (np.array_equal(gb, rb[off:off + bud]) and np.array_equal(gf, rfs[off:off + bud])):
                print(f"  iter {m}: gpu buckets {gb[:12]} f {gf[:12]}\n          ref buckets {rb[off:off+bud][:12]} f {rfs[off:off+bud][:12]} status {tr['sel_status'][off:off+bud][:12]}")
                break
            off += bud


if __name__ == "__main__":
    print("devices", M.device_count(), flush=True)
    check_window(1024, 32, 1e-6)
    check_window(8192, 256, 1e-6)
    check_window(1 << 16, 256, 1e-8)
    check_window(1 << 16, 32, 1e-8)
    check_sfft(1 << 12, 10, 1)
    check_sfft(1 << 16, 50, 1)
    check_sfft(1 << 16, 50, 2)
    check_sfft(1 << 16, 50, 3, dtype=np.complex64)
    check_sfft(1 << 18, 100, 4, snr=20.0)
    check_sfft(1 << 18, 100, 5, snr=20.0, l=8, q=2.0)
    check_sfft(1 << 20, 100, 1, snr=20.0)
