"""Times the host-input path of Plan.execute on the C4 workload: sparse ingest
(validating and ASSUME_VALID) and the dense whole-signal H2D path.  Prints
one JSON line.  Thread count / chunk come from MSFFT_INGEST_THREADS /
MSFFT_INGEST_CHUNK."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_05698_b200 as M  # noqa: E402
from paper_2011_05698_b200.workloads import algo_seed, make_batch, signal_seed  # noqa: E402

B = int(os.environ.get("PROBE_BATCH", "1024"))
n, k, delta = 1 << 22, 64, 1e-6
seeds = [signal_seed(0xC4C40000, i) for i in range(B)]
aseeds = np.array([algo_seed(s) for s in seeds], dtype=np.uint64)
x, _ = make_batch(n, k, seeds, 25.0, torch.device("cuda", 0), "complex64")
xh = torch.empty((B, n), dtype=torch.complex64, pin_memory=True)
xh.copy_(x)
del x
torch.cuda.synchronize()
res = {"batch": B, "threads": os.environ.get("MSFFT_INGEST_THREADS", str(os.cpu_count())),
       "chunk": os.environ.get("MSFFT_INGEST_CHUNK", "128")}


def timed(plan, reps=3, **kw):
    plan.execute(xh, aseeds, **kw)
    t0 = time.perf_counter()
    for _ in range(reps):
        plan.execute(xh, aseeds, **kw)
    return (time.perf_counter() - t0) / reps * 1e3


plan = M.Plan(n, k, M.MultiscaleConfig(), delta, "complex64", 0)
res["ingest_samples"] = plan.ingest_samples_per_signal
per = []
for _ in range(8):
    t0 = time.perf_counter()
    plan.execute(xh, aseeds)
    per.append(round((time.perf_counter() - t0) * 1e3, 1))
res["sparse_validate_ms_per_call"] = per
res["sparse_validate_ms"] = min(per[-4:])
res["sparse_assume_valid_ms"] = timed(plan, assume_valid=True)
if os.environ.get("PROBE_DENSE", "1") == "1":
    os.environ["MSFFT_SPARSE_INGEST"] = "0"
    dense = M.Plan(n, k, M.MultiscaleConfig(), delta, "complex64", 0)
    res["dense_validate_ms"] = timed(dense, reps=2)
print(json.dumps(res))
