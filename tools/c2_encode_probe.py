"""C2 (N=2^20, K=100, 20 dB) at (l, q) = (4, 2): one plan, a validating
call, then serial executes -- for an ncu look at the encode launch."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2011_05698_b200 as M  # noqa: E402
from helpers import make_signal  # noqa: E402
from oracle import available, load  # noqa: E402

R = load("reference" if available("reference") else "port")
x = make_signal(R, dict(gen="ref", n=1 << 20, k=100, seed=1, snr=20.0))
l, q = (int(sys.argv[1]), float(sys.argv[2])) if len(sys.argv) > 2 else (4, 2.0)
plan = M.Plan(1 << 20, 100, M.MultiscaleConfig(l, q), 1e-6, "complex128", 0)
xd = torch.as_tensor(x.reshape(1, -1)).to("cuda")
seeds = np.array([M.splitmix64(1 ^ 0x53)], np.uint64)
plan.execute(xd, seeds)
for _ in range(2):
    _, _, _, ms = plan.execute(xd, seeds, assume_valid=True, stage_times=True, serial=True)
    print("ms", round(ms, 4), [round(t, 4) for t in plan.stage_times()], flush=True)
