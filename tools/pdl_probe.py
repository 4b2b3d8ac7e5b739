"""Per-step time of the asynchronous C4 loop on the legacy default stream vs
a dedicated stream, with and without programmatic dependent launch (set
MSFFT_PDL before running)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_05698_b200 as M  # noqa: E402
from paper_2011_05698_b200.workloads import algo_seed, make_batch, signal_seed  # noqa: E402

B, n, k = 1024, 1 << 22, 64
dev = torch.device("cuda", 0)
seeds = [signal_seed(0xC4C40000, i) for i in range(B)]
a = np.array([algo_seed(s) for s in seeds], dtype=np.uint64)
sets = (a, a ^ np.uint64(0x9E3779B97F4A7C15))
x, _ = make_batch(n, k, seeds, 25.0, dev, "complex64")
plan = M.Plan(n, k, M.MultiscaleConfig(), 1e-6, "complex64", 0)
out = (torch.empty((B, k), dtype=torch.int64, device=dev),
       torch.empty((B, k), dtype=torch.complex128, device=dev),
       torch.empty((B,), dtype=torch.int64, device=dev))
plan.execute(x, a, out=out)
for name, stream in (("legacy", torch.cuda.default_stream(dev)), ("dedicated", torch.cuda.Stream(dev))):
    with torch.cuda.stream(stream):
        h = stream.cuda_stream
        for i in range(4):
            plan.execute(x, sets[i & 1], out=out, assume_valid=True, stream=h, async_=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(20):
            plan.execute(x, sets[i & 1], out=out, assume_valid=True, stream=h, async_=True)
        e1.record(stream)
        torch.cuda.synchronize()
        plan.sync(h)
        print(f"PDL={os.environ.get('MSFFT_PDL', '1')} {name:9s} {e0.elapsed_time(e1) / 20:.3f} ms/step",
              flush=True)
