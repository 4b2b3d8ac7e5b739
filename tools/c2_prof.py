import sys, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, torch
import paper_2011_05698_b200 as M
from helpers import make_signal
from oracle import available, load
R = load("reference" if available("reference") else "port")
x = make_signal(R, dict(gen="ref", n=1 << 20, k=100, seed=1, snr=20.0))
for l, q in ((4, 2.0), (8, 1.0)):
    plan = M.Plan(1 << 20, 100, M.MultiscaleConfig(l, q), 1e-6, "complex128", 0)
    xd = torch.as_tensor(x.reshape(1, -1)).to("cuda")
    seeds = np.array([M.splitmix64(1 ^ 0x53)], np.uint64)
    plan.execute(xd, seeds)
    print("== l q", l, q, flush=True)
    _, _, _, ms = plan.execute(xd, seeds, assume_valid=True, stage_times=True, serial=True)
    print("ms", ms, plan.stage_times(), flush=True)
