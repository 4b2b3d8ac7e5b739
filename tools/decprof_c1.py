"""Per-phase decode cycles (clock64 marks of decode_body.cuh, diagnostic
build tools/build_variant.py decprof -DMSFFT_DECODE_PROFILE) for one C1 and
one C4 signal:  MSFFT_B200_LIB=tools/variants/lib_decprof.so python tools/decprof_c1.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_05698_b200 as M  # noqa: E402
from paper_2011_05698_b200.workloads import make_signal_np  # noqa: E402

for n, k, delta, snr in ((1 << 16, 50, 1e-8, None), (1 << 22, 64, 1e-6, 25.0)):
    x, _, _ = make_signal_np(n, k, 1, snr, "complex128")
    plan = M.Plan(n, k, M.MultiscaleConfig(), delta, "complex128")
    for rep in range(2):
        f, c, cnt, ms = plan.execute(x[None, :], [7], serial=True, stage_times=True)
        print(f"n={n} k={k} rep={rep} device_ms={ms:.4f} stages={plan.stage_times()}", flush=True)
