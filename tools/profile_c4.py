"""C4 batch for profiling: generate, plan, execute `--reps` times (device
resident, ASSUME_VALID after the first validating call).  Run it plain first,
then under ncu (see profiles/README.md)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_05698_b200 as M  # noqa: E402
from paper_2011_05698_b200.workloads import algo_seed, make_batch, signal_seed  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=1024)
ap.add_argument("--log2n", type=int, default=22)
ap.add_argument("--k", type=int, default=64)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--no-stages", action="store_true")
ap.add_argument("--serial", action="store_true", help="separate encode / decode launches")
ap.add_argument("--validate", action="store_true",
                help="every rep validating (the fused_val_kernel launch)")
a = ap.parse_args()
n, k, B = 1 << a.log2n, a.k, a.batch
dev = torch.device("cuda", 0)
seeds = [signal_seed(0xC4C40000, i) for i in range(B)]
aseeds = np.array([algo_seed(s) for s in seeds], dtype=np.uint64)
x, _ = make_batch(n, k, seeds, 25.0, dev, "complex64")
plan = M.Plan(n, k, M.MultiscaleConfig(), 1e-6, "complex64", 0)
out = (torch.empty((B, k), dtype=torch.int64, device=dev),
       torch.empty((B, k), dtype=torch.complex128, device=dev),
       torch.empty((B,), dtype=torch.int64, device=dev))
sh = torch.cuda.current_stream().cuda_stream
for r in range(a.reps):
    _, _, _, ms = plan.execute(x, aseeds, out=out, assume_valid=r > 0 and not a.validate, stream=sh,
                               stage_times=not a.no_stages, serial=a.serial)
    print(f"rep {r}: {ms:.3f} ms  stages {plan.stage_times()}", flush=True)

if a.reps > 2:
    import statistics
    import json
    print("SUMMARY " + json.dumps({"lib": os.environ.get("MSFFT_B200_LIB", "product"),
                                   "serial": a.serial}), flush=True)
