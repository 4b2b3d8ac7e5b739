"""Validating C4 step (1024 x N=2^22, K=64, c64, device resident) under
environment variants of the validating fused launch (engine.cu val_for):
median CUDA-event ms of `--reps` validating execute calls per variant, all
variants in one process on the same batch.  Usage:
    python tools/val_sweep.py "MSFFT_VAL_FUSED=0" "MSFFT_VAL_ITEM_KB=512" ...
(an argument holds space-separated KEY=VALUE pairs; "" = defaults)."""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_05698_b200 as M  # noqa: E402
from paper_2011_05698_b200.workloads import algo_seed, make_batch, signal_seed  # noqa: E402

KEYS = ("MSFFT_VAL_FUSED", "MSFFT_VAL_CHUNK_MB", "MSFFT_VAL_ITEM_KB", "MSFFT_VAL_DLAG",
        "MSFFT_VAL_ELAG", "MSFFT_VAL_DEBUG", "MSFFT_VAL_EFIRST",
        "MSFFT_VAL_POLICY", "MSFFT_VAL_EOFF", "MSFFT_VAL_SMEM_KB", "MSFFT_VAL_SPLIT")
reps = int(os.environ.get("REPS", "7"))
n, k, B = 1 << 22, 64, int(os.environ.get("BATCH", "1024"))
dev = torch.device("cuda", 0)
seeds = [signal_seed(0xC4C40000, i) for i in range(B)]
aseeds = np.array([algo_seed(s) for s in seeds], dtype=np.uint64)
x, _ = make_batch(n, k, seeds, 25.0, dev, "complex64")
out = (torch.empty((B, k), dtype=torch.int64, device=dev),
       torch.empty((B, k), dtype=torch.complex128, device=dev),
       torch.empty((B,), dtype=torch.int64, device=dev))
sh = torch.cuda.current_stream().cuda_stream
ref = None
for arg in sys.argv[1:] or [""]:
    for key in KEYS:
        os.environ.pop(key, None)
    for kv in arg.split():
        key, v = kv.split("=")
        os.environ[key] = v
    plan = M.Plan(n, k, M.MultiscaleConfig(), 1e-6, "complex64", 0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for r in range(reps + 1):
        e0.record()
        plan.execute(x, aseeds, out=out, stream=sh)
        e1.record()
        e1.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1))
    same = None
    if "MSFFT_VAL_DEBUG" not in arg:
        cur = [t.cpu().numpy().copy() for t in out]
        if ref is None:
            ref = cur
        same = all(np.array_equal(a, b) for a, b in zip(ref, cur))
    print(json.dumps({"env": arg, "launches": plan.launches(B), "median_ms": statistics.median(ts),
                      "min_ms": min(ts), "same_as_first": same}), flush=True)
    del plan
