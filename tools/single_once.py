"""One small config, executed --reps times (device-resident input, the first
call validates): a target for ncu captures of the single-signal kernels.

    python tools/single_once.py C1 [--serial] [--reps 4]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_05698_b200 as M  # noqa: E402
from paper_2011_05698_b200.workloads import make_signal_np  # noqa: E402

CFG = {"C1": (1 << 16, 50, 16, 1.0, 1e-8, "complex128", None),
       "C4one": (1 << 22, 64, 16, 1.0, 1e-6, "complex64", 25.0),
       "C2_4_2": (1 << 20, 100, 4, 2.0, 1e-6, "complex128", 20.0),
       "C2_8_1": (1 << 20, 100, 8, 1.0, 1e-6, "complex128", 20.0)}
ap = argparse.ArgumentParser()
ap.add_argument("cfg", choices=sorted(CFG))
ap.add_argument("--serial", action="store_true")
ap.add_argument("--reps", type=int, default=4)
a = ap.parse_args()
n, k, l, q, delta, dtype, snr = CFG[a.cfg]
x = make_signal_np(n, k, 3, snr, dtype)[0].astype(dtype)
plan = M.Plan(n, k, M.MultiscaleConfig(l, q), delta, dtype)
for r in range(a.reps):
    ms = plan.execute(x[None, :], [7], assume_valid=r > 0, serial=a.serial)[3]
    print(f"rep {r}: {ms:.4f} ms", flush=True)
