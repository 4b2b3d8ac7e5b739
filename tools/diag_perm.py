"""Diagnostic: batch results vs single-signal and permuted-batch results."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_05698_b200 as M  # noqa: E402
from paper_2011_05698_b200.workloads import algo_seed, make_batch, signal_seed  # noqa: E402

N, K = 1 << 22, 64
for B in (int(a) for a in sys.argv[1:] or ["64", "1024"]):
    seeds = [signal_seed(0x7E57, i) for i in range(B)]
    s = np.array([algo_seed(v) for v in seeds], dtype=np.uint64)
    x, _ = make_batch(N, K, seeds, 25.0, torch.device("cuda", 0), "complex64")
    plan = M.Plan(N, K, M.MultiscaleConfig(), 1e-6, "complex64")

    def run(xx, ss):
        b = xx.shape[0]
        out = (torch.empty((b, K), dtype=torch.int64, device="cuda"),
               torch.empty((b, K), dtype=torch.complex128, device="cuda"),
               torch.empty((b,), dtype=torch.int64, device="cuda"))
        plan.execute(xx, ss, out=out)
        return [o.cpu().numpy() for o in out]

    f1, c1, n1 = run(x, s)
    f1b, c1b, n1b = run(x, s)
    print(B, "repeat equal:", np.array_equal(f1, f1b) and np.array_equal(c1, c1b), flush=True)
    bad_single = []
    for i in list(range(min(B, 40))):
        fs, cs, ns = run(x[i:i + 1], s[i:i + 1])
        if not (np.array_equal(fs[0], f1[i]) and np.array_equal(cs[0], c1[i])):
            bad_single.append(i)
    print(B, "single-vs-batch mismatches:", bad_single, flush=True)
    perm = np.random.default_rng(5).permutation(B)
    xp = torch.empty_like(x)
    for i, p in enumerate(perm):
        xp[i].copy_(x[int(p)])
    f2, c2, n2 = run(xp, s[perm])
    badp = [i for i in range(B) if not (np.array_equal(f2[i], f1[perm[i]]) and np.array_equal(c2[i], c1[perm[i]]))]
    print(B, "perm mismatches:", len(badp), badp[:20], flush=True)
    if badp:
        i = badp[0]
        print(" f2", f2[i][:10], "\n f1", f1[perm[i]][:10])
        fs, cs, _ = run(x[perm[i]:perm[i] + 1], s[perm[i]:perm[i] + 1])
        print(" single equals batch:", np.array_equal(fs[0], f1[perm[i]]), " single equals perm:", np.array_equal(fs[0], f2[i]))
    del x, xp
    torch.cuda.empty_cache()
