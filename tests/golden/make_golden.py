"""Generates tests/golden/*.json from the reference itself (oracle/_ref, the
reference library compiled from /root/reference by oracle/Makefile).

Run in the build container, where /root/reference exists:
    make -C oracle ref && python tests/golden/make_golden.py [names...]
Signals are stored as recipes (generator + seeds), never as samples:
  gen "ref": the reference's own generate_test_signal + add_awgn with the
             bench's seed derivation (proj/src/bench.cpp:115-120);
  gen "np":  paper_2011_05698_b200.workloads.make_signal_np (numpy only);
  gen "zero": all-zero signal.
Floats are stored with float.hex() so comparisons can be bit-exact.
"""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import json
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from oracle import load  # noqa: E402
from paper_2011_05698_b200 import splitmix64  # noqa: E402
from paper_2011_05698_b200.workloads import make_signal_np  # noqa: E402


def hx(v):
    return float(v).hex()


def make_signal(o, rec):
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


def run_case(o, rec):
    x = make_signal(o, rec).astype(np.complex128)
    out = dict(rec)
    try:
        t = time.time()
        r = o.sfft4(x, rec["k"], rec["l"], rec["q"], rec["algo_seed"], rec["delta"])
        out["result"] = {"f": [int(v) for v in r.f],
                         "c": [[hx(v.real), hx(v.imag)] for v in r.c],
                         "stats": {kk: vv for kk, vv in r.stats.items() if kk != "runtime_ms"}}
        out["ref_runtime_ms"] = r.stats["runtime_ms"]
        out["wall_s"] = time.time() - t
    except Exception as e:  # noqa: BLE001
        out["error"] = {"kind": getattr(e, "kind", "other"), "msg": str(e)}
    return out


def case(gen, n, k, seed, snr, l=16, q=1.0, dtype="complex128", **kw):
    delta = 1e-6 if snr is not None else 1e-8
    rec = dict(gen=gen, n=n, k=k, seed=seed, snr=snr, l=l, q=q, dtype=dtype, delta=delta,
               algo_seed=splitmix64(seed ^ 0x53))
    rec.update(kw)
    return rec


def known_answers(o):
    d = {}
    d["tau_schedule"] = [[32.0, 8192, o.tau_schedule(32.0, 8192)],
                         [256.0, 1 << 16, o.tau_schedule(256.0, 1 << 16)],
                         [3.0, 1 << 20, o.tau_schedule(3.0, 1 << 20)]]
    d["stage_count"] = [[L, l, q, o.stage_count(L, l, q)]
                        for L in (2, 16, 32, 256, 2048, 16384, 131072)
                        for (l, q) in ((16, 1.0), (8, 2.0), (4, 1.0), (8, 4.0), (16, 0.0))]
    ok, qm = o.check_parameter_bounds(0.3, 4)
    d["check_parameter_bounds"] = [[0.3, 4, ok, hx(qm)]]
    d["mod_inverse"] = [[s, n, o.mod_inverse(s, n)] for (s, n) in
                        ((1, 64), (3, 8), (5, 16), (12345, 1 << 16), (987654321, 1 << 30))]
    d["bucket_of"] = [[u, L, b, o.bucket_of(u, L, b)] for (u, L, b) in
                      ((16, 32, 256), (15, 32, 256), (8192 - 16, 32, 256), (8192 - 17, 32, 256))]
    s, si = o.random_params(1024, 99, 8)
    d["random_params"] = {"n": 1024, "seed": 99, "sigma": [int(v) for v in s],
                          "sigma_inv": [int(v) for v in si]}
    s, si = o.random_params(1 << 22, 12345, 8)
    d["random_params_big"] = {"n": 1 << 22, "seed": 12345, "sigma": [int(v) for v in s],
                              "sigma_inv": [int(v) for v in si]}
    d["splitmix64"] = [[v, o.splitmix64(v)] for v in (0, 1, 0x51, 0x53, 2**63 + 5)]
    d["initial_bucket_count"] = [[n, k, dl, o.initial_bucket_count(n, k, dl)] for (n, k, dl) in
                                 ((1 << 16, 50, 1e-8), (1 << 20, 100, 1e-6), (1 << 22, 64, 1e-6),
                                  (8192, 50, 1e-8), (4096, 10, 1e-8))]
    return d


def windows(o):
    specs = [(1024, 32, 1e-6), (4096, 64, 1e-6), (4096, 64, 1e-8), (8192, 256, 1e-6),
             (8192, 64, 1e-8), (16384, 128, 1e-8), (65536, 256, 1e-6), (65536, 512, 1e-6),
             (1 << 16, 256, 1e-8), (1 << 16, 128, 1e-8), (1 << 16, 64, 1e-8), (1 << 16, 32, 1e-8),
             (1 << 20, 512, 1e-6), (1 << 20, 32, 1e-6)]
    bad = [(8192, 256, 1e-8), (8192, 2048, 1e-6), (8192, 3, 1e-6), (8192, 64, 0.5),
           (8192, 64, 0.0), (1000, 10, 1e-6), (8, 4, 1e-6)]
    out = {"ok": [], "error": []}
    for n, b, dl in specs:
        w, g = o.window(n, b, dl)
        L = n // b
        offs = [0, 1, L // 2, L, 3 * L // 2, -1, -(L // 2), -(3 * L // 2)]
        resp = o.response_at(n, b, dl, offs)
        out["ok"].append({"n": n, "b": b, "delta": dl, "w": w,
                          "taps_sha256": hashlib.sha256(g.astype("<f8").tobytes()).hexdigest(),
                          "taps_head": [hx(v) for v in g[:4]],
                          "taps_mid": hx(g[(w - 1) // 2]),
                          "response": [[int(a), hx(v)] for a, v in zip(offs, resp)]})
    for n, b, dl in bad:
        try:
            o.window(n, b, dl)
            out["error"].append({"n": n, "b": b, "delta": dl, "msg": None})
        except Exception as e:  # noqa: BLE001
            out["error"].append({"n": n, "b": b, "delta": dl, "msg": str(e)})
    return out


def small_cases():
    cs = []
    for seed in (1, 2, 3, 4, 5):
        cs.append(case("ref", 1 << 16, 50, seed, None))                 # C1
    for l in (2, 4, 8):
        for q in (1.0, 2.0, 4.0):
            cs.append(case("ref", 1 << 20, 100, 1, 20.0, l=l, q=q))      # C2 sweep
    cs.append(case("ref", 1 << 20, 100, 1, 20.0))                        # C2 default l,q
    cs += [case("np", 1 << 12, 10, 7, None), case("np", 1 << 12, 1, 8, None),
           case("np", 64, 2, 9, None), case("np", 16, 1, 10, None), case("np", 1 << 13, 50, 11, None),
           case("np", 1 << 16, 50, 12, None, dtype="complex64"),
           case("np", 1 << 18, 100, 13, 20.0, l=8, q=2.0),
           case("np", 1 << 18, 100, 14, 20.0, l=4, q=1.0),
           case("np", 1 << 14, 200, 15, 10.0),
           case("zero", 1 << 12, 10, 16, None),
           case("np", 1 << 12, 600, 17, None),        # K > n/8: invalid
           case("np", 1 << 12, 0, 18, None),          # K = 0: invalid
           case("np", 1 << 16, 50, 19, None, l=16, q=20.0),  # l/(q+1) < 1: invalid
           case("np", 1 << 12, 10, 20, 30.0, delta_override=0.5)]
    for c in cs:
        if "delta_override" in c:
            c["delta"] = c.pop("delta_override")
    return cs


def c4_cases():
    return [case("np", 1 << 22, 64, s, 25.0, dtype="complex64") for s in (101, 102, 103, 104)]


def c3_cases():
    n, b1 = 1 << 24, 4096
    return [case("np", n, 1000, 301, 30.0, dtype=dt, magnitude="uniform_0.5_2",
                 min_sep=4 * n // b1) for dt in ("complex128", "complex64")]


def big_cases():
    """C5-law signals at sizes the reference finishes in minutes: large b
    (8192), budget (2000) and accumulated list (~4000) -- the decode's
    radix-sort paths."""
    return [case("np", 1 << 20, 2000, 501, 20.0, magnitude="loguniform_0.1_10"),
            case("np", 1 << 19, 1200, 502, 20.0, dtype="complex64",
                 magnitude="loguniform_0.1_10")]


def c5_case():
    """BASELINE.json configs[4]: N=2^27, K=10^4, complex128, |c| log-uniform
    [0.1, 10], 20 dB (delta 1e-6, l=16, q=1)."""
    return case("np", 1 << 27, 10000, 505, 20.0, magnitude="loguniform_0.1_10")


def c3_more_cases():
    n, b1 = 1 << 24, 4096
    return [case("np", n, 1000, s, 30.0, dtype=dt, magnitude="uniform_0.5_2",
                 min_sep=4 * n // b1) for s in (302, 303) for dt in ("complex128", "complex64")]


def bucket_schedule(o, n, k, delta):
    b = o.initial_bucket_count(n, k, delta)
    bs = []
    for _ in range(int(math.ceil(math.log2(k))) + 2):
        if b not in bs:
            bs.append(b)
        b = b // 2 if b > 32 else b
    return bs


def prewarm(o, n, k, delta, workers=None):
    """Designs every window of the transform's schedule in parallel threads
    (the reference's process cache, window.cpp:179-193, designs outside its
    lock).  At n=2^27 one design holds ~5.5 GB, so `workers` bounds memory."""
    bs = bucket_schedule(o, n, k, delta)
    with cf.ThreadPoolExecutor(workers or len(bs)) as ex:
        list(ex.map(lambda bb: o.window(n, bb, delta, False), sorted(bs, reverse=True)))


def window_shas(o, n, k, delta):
    out = []
    for b in bucket_schedule(o, n, k, delta):
        w, g = o.window(n, b, delta)
        out.append({"n": n, "b": b, "delta": delta, "w": w,
                    "taps_sha256": hashlib.sha256(g.astype("<f8").tobytes()).hexdigest(),
                    "taps_mid": hx(g[(w - 1) // 2])})
        del g
    return out


def dump(name, obj):
    path = os.path.join(HERE, name + ".json")
    with open(path, "w") as f:
        json.dump(obj, f, indent=1)
    print("wrote", path, flush=True)


def main(names):
    o = load("reference")
    if "known" in names:
        dump("known_answers", known_answers(o))
    if "windows" in names:
        dump("windows", windows(o))
    if "small" in names:
        dump("sfft4_small", [run_case(o, c) for c in small_cases()])
    if "c4" in names:
        prewarm(o, 1 << 22, 64, 1e-6)
        dump("sfft4_c4", [run_case(o, c) for c in c4_cases()])
    if "big" in names:
        for c in big_cases():
            prewarm(o, c["n"], c["k"], c["delta"])
        dump("sfft4_big", [run_case(o, c) for c in big_cases()])
    if "c3" in names:
        prewarm(o, 1 << 24, 1000, 1e-6)
        dump("sfft4_c3", [run_case(o, c) for c in c3_cases()])
    if "c3more" in names:
        prewarm(o, 1 << 24, 1000, 1e-6)
        dump("sfft4_c3_more", [run_case(o, c) for c in c3_more_cases()])
    if "c5" in names:
        # ~1 h of window design (6 concurrent, ~5.5 GB each) then ~1-1.5 h of
        # single-threaded sfft4; run in the background.
        c = c5_case()
        t = time.time()
        prewarm(o, c["n"], c["k"], c["delta"], workers=6)
        wins = window_shas(o, c["n"], c["k"], c["delta"])
        dump("sfft4_c5_windows", {"design_wall_s": time.time() - t, "windows": wins})
        res = run_case(o, c)
        res["windows"] = wins
        dump("sfft4_c5", res)


if __name__ == "__main__":
    main(sys.argv[1:] or ["known", "windows", "small"])
