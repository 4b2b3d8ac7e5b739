"""Host-side cost of one small-batch call: wall time of msfft_execute with
MSFFT_FLAG_ASYNC (returns once enqueued) against the device-event time of a
synchronous call, for the single-signal configs.

    python tools/host_overhead.py"""
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_05698_b200 as M  # noqa: E402
from paper_2011_05698_b200.workloads import make_signal_np  # noqa: E402

dev = torch.device("cuda", 0)
for name, n, k, l, q, delta, dtype, snr in (("C1", 1 << 16, 50, 16, 1.0, 1e-8, "complex128", None),
                                             ("C4one", 1 << 22, 64, 16, 1.0, 1e-6, "complex64", 25.0)):
    x = torch.as_tensor(make_signal_np(n, k, 3, snr, dtype)[0].astype(dtype).reshape(1, -1)).to(dev)
    plan = M.Plan(n, k, M.MultiscaleConfig(l, q), delta, dtype)
    out = (torch.empty((1, k), dtype=torch.int64, device=dev),
           torch.empty((1, k), dtype=torch.complex128, device=dev),
           torch.empty((1,), dtype=torch.int64, device=dev))
    plan.execute(x, [7], out=out)
    ev = [plan.execute(x, [7], out=out, assume_valid=True)[3] for _ in range(20)]
    enq = []
    for i in range(200):
        t0 = time.perf_counter_ns()
        plan.execute(x, [7], out=out, assume_valid=True, async_=True)
        enq.append((time.perf_counter_ns() - t0) / 1000)
        if i % 10 == 9:
            plan.sync()
    plan.sync()
    t0 = time.perf_counter_ns()
    for i in range(200):
        plan.execute(x, [7], out=out, assume_valid=True, async_=True)
    plan.sync()
    per = (time.perf_counter_ns() - t0) / 1000 / 200
    print(f"{name}: event ms median {statistics.median(ev):.4f}; async enqueue us median "
          f"{statistics.median(enq):.1f}; back-to-back async per call {per:.1f} us", flush=True)
