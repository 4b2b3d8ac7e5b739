"""Per-config timing table (BASELINE.json configs C1-C5) on one B200: GPU time
per transform (device-resident input, validated once, CUDA events around
msfft_execute, median of reps after a warm-up; per-stage times from the
serial path) beside the reference's own sfft4 on the box's CPU (its internal
timer, TransformStats::runtime_ms, one thread) on the same input, with the
parity check.  C5's reference run takes hours (window design alone > 22 min
per window) and is skipped.  Prints one JSON line per config and a summary.

    python tools/configs_table.py [--no-ref] [C1 C2 C3 C4 C5]

--no-ref times the GPU side only (parity is then not checked here).
"""
import json
import math
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2011_05698_b200 as M  # noqa: E402
from helpers import make_signal, parity, prewarm_windows  # noqa: E402
from oracle import available, load  # noqa: E402
from paper_2011_05698_b200 import splitmix64  # noqa: E402
from paper_2011_05698_b200.workloads import algo_seed, make_batch, signal_seed  # noqa: E402

R = load("reference" if available("reference") else "port")
dev = torch.device("cuda", 0)
TOL = {"complex128": 1e-9, "complex64": 1e-4}


def gpu_time(x_host, k, l, q, seed, delta, dtype, reps=7):
    n = x_host.shape[-1]
    plan = M.Plan(n, k, M.MultiscaleConfig(l, q), delta, dtype, 0)
    xd = torch.as_tensor(x_host.reshape(1, -1)).to(dev)
    seeds = np.array([seed], np.uint64)
    out = (torch.empty((1, k), dtype=torch.int64, device=dev),
           torch.empty((1, k), dtype=torch.complex128, device=dev),
           torch.empty((1,), dtype=torch.int64, device=dev))
    plan.execute(xd, seeds, out=out)  # validating call + warm-up
    ms, msv = [], []
    for _ in range(reps):
        _, _, _, t = plan.execute(xd, seeds, out=out, assume_valid=True)
        ms.append(t)
        _, _, _, t = plan.execute(xd, seeds, out=out)  # validates every sample, as sfft4.cpp:133
        msv.append(t)
    plan.execute(xd, seeds, out=out, assume_valid=True, stage_times=True, serial=True)
    stages = plan.stage_times()
    f, c, cnt = out[0].cpu().numpy(), out[1].cpu().numpy(), int(out[2].cpu().numpy()[0])
    return statistics.median(ms), statistics.median(msv), stages, f[0, :cnt], c[0, :cnt]


NO_REF = "--no-ref" in sys.argv


def cell(name, x, k, l, q, seed, delta, dtype, ref=True, golden=None):
    ref = ref and not NO_REF
    row = {"config": name, "n": int(x.shape[-1]), "k": k, "l": l, "q": q, "dtype": dtype}
    try:
        g_ms, g_ms_val, stages, f, c = gpu_time(x, k, l, q, seed, delta, dtype)
    except Exception as e:  # noqa: BLE001  (invalid (l, q) cells raise like the reference)
        row["gpu_error"] = str(e)
        g_ms = None
    if g_ms is not None:
        row.update(gpu_ms=g_ms, gpu_ms_validating=g_ms_val,
                   gpu_stage_ms={"encode": stages[0], "bucket_fft": stages[1],
                                 "decode": stages[2]})
    if golden is not None and g_ms is not None:
        # the reference's result on the same bytes from a committed fixture
        from helpers import golden_result
        gf, gc, _ = golden_result(golden)
        same, err, _ = parity(gf, gc, f, c, k, delta, TOL[dtype])
        row.update(ref_ms=golden["ref_runtime_ms"], ref_source="tests/golden/sfft4_c5.json",
                   speedup=golden["ref_runtime_ms"] / g_ms, support_identical=bool(same),
                   max_rel_err=err)
    if ref:
        try:
            prewarm_windows(R, int(x.shape[-1]), k, delta)  # untimed, as sfft4.cpp:146-154
            r = R.sfft4(x.astype(np.complex128), k, l, q, seed, delta)
            row["ref_ms"] = r.stats["runtime_ms"]
            if g_ms is not None:
                same, err, _ = parity(r.f, r.c, f, c, k, delta, TOL[dtype])
                row.update(speedup=row["ref_ms"] / g_ms, support_identical=bool(same),
                           max_rel_err=err)
        except Exception as e:  # noqa: BLE001
            row["ref_error"] = str(e)
    print(json.dumps(row), flush=True)
    return row


def main(names):
    rows = []
    if "C1" in names:
        for s in (1, 2, 3):
            rec = dict(gen="ref", n=1 << 16, k=50, seed=s, snr=None)
            x = make_signal(R, rec)
            rows.append(cell("C1", x, 50, 16, 1.0, splitmix64(s ^ 0x53), 1e-8, "complex128"))
    if "C2" in names:
        rec = dict(gen="ref", n=1 << 20, k=100, seed=1, snr=20.0)
        x = make_signal(R, rec)
        for l in (2, 4, 8):
            for q in (1.0, 2.0, 4.0):
                rows.append(cell("C2", x, 100, l, q, splitmix64(1 ^ 0x53), 1e-6, "complex128"))
    if "C3" in names:
        for dt in ("complex128", "complex64"):
            n, b1 = 1 << 24, 4096
            rec = dict(gen="np", n=n, k=1000, seed=301, snr=30.0, dtype=dt,
                       magnitude="uniform_0.5_2", min_sep=4 * n // b1)
            x = make_signal(R, rec)
            rows.append(cell("C3", x, 1000, 16, 1.0, splitmix64(301 ^ 0x53), 1e-6, dt))
    if "C4" in names:
        rec = dict(gen="np", n=1 << 22, k=64, seed=101, snr=25.0, dtype="complex64")
        x = make_signal(R, rec)
        rows.append(cell("C4 (one signal)", x, 64, 16, 1.0, splitmix64(101 ^ 0x53), 1e-6,
                         "complex64"))
    if "C5" in names:
        gpath = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                             "tests", "golden", "sfft4_c5.json")
        if os.path.exists(gpath):  # the reference ran on these bytes (make_golden.py c5)
            rec = json.load(open(gpath))
            x = make_signal(R, rec)
            rows.append(cell("C5", x, rec["k"], rec["l"], rec["q"], rec["algo_seed"],
                             rec["delta"], "complex128", ref=False, golden=rec))
        else:
            s = signal_seed(0xC5C50000, 0)
            xb, _ = make_batch(1 << 27, 10000, [s], 20.0, dev, "complex128",
                               magnitude="loguniform_0.1_10", chunk=1)
            x = xb[0].cpu().numpy()
            del xb
            torch.cuda.empty_cache()
            rows.append(cell("C5", x, 10000, 16, 1.0, algo_seed(s), 1e-6, "complex128", ref=False))
    print("SUMMARY " + json.dumps(rows))


if __name__ == "__main__":
    main([a for a in sys.argv[1:] if not a.startswith("--")] or ["C1", "C2", "C3", "C4", "C5"])
