import os, sys
sys.path.insert(0, os.getcwd())
import paper_2011_05698_b200 as M
from paper_2011_05698_b200.workloads import make_signal_np
for (n, k, l, q, d, snr) in ((1 << 20, 100, 4, 2.0, 1e-6, 20.0), (1 << 16, 50, 16, 1.0, 1e-8, None)):
    x = make_signal_np(n, k, 3, snr, "complex128")[0]
    plan = M.Plan(n, k, M.MultiscaleConfig(l, q), d, "complex128")
    for rep in range(2):
        plan.execute(x[None, :], [7], serial=True)
        print("---", n, k, l, q, rep, flush=True)
