"""C3 (N=2^24, K=1000, min-separated support, 30 dB) for per-stage
profiling: one plan, a validating call, then --reps calls with ASSUME_VALID
on the serial path (encode -> bucket FFTs -> decode).  Run plain first, then
under ncu (see profiles/README.md)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_05698_b200 as M  # noqa: E402
from paper_2011_05698_b200 import splitmix64  # noqa: E402
from paper_2011_05698_b200.workloads import make_signal_np  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dtype", default="complex128")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--no-stages", action="store_true",
                help="the production path (no per-stage events, encode/decode overlapped)")
a = ap.parse_args()
n, k = 1 << 24, 1000
x, _, _ = make_signal_np(n, k, 301, 30.0, a.dtype, "uniform_0.5_2", 4 * n // 4096)
dev = torch.device("cuda", 0)
xd = torch.as_tensor(x.astype(a.dtype).reshape(1, -1)).to(dev)
plan = M.Plan(n, k, M.MultiscaleConfig(), 1e-6, a.dtype, 0)
seeds = np.array([splitmix64(301 ^ 0x53)], np.uint64)
out = (torch.empty((1, k), dtype=torch.int64, device=dev),
       torch.empty((1, k), dtype=torch.complex128, device=dev),
       torch.empty((1,), dtype=torch.int64, device=dev))
plan.execute(xd, seeds, out=out)
if os.environ.get("MSFFT_PROFILE_AFTER_PLAN"):
    torch.cuda.synchronize()
    torch.cuda.profiler.start()  # ncu --profile-from-start off: skip window design
for r in range(a.reps):
    st = not a.no_stages
    _, _, _, ms = plan.execute(xd, seeds, out=out, assume_valid=True, stage_times=st, serial=st)
    print(f"rep {r}: {ms:.3f} ms  stages {plan.stage_times()}", flush=True)
