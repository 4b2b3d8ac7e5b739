"""Config 5 (BASELINE.json configs[4]): one N=2^27, K=10000, complex128 signal,
log-uniform magnitudes [0.1, 10], AWGN 20 dB.  Runs sfft4 on the GPU through
the batched plan (window design included in plan creation), then checks the
size-independent properties available without a reference run (the CPU
reference needs hours at this size): determinism, exact doubling, support
size and ordering.  Prints one JSON line."""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_05698_b200 as M  # noqa: E402
from paper_2011_05698_b200.workloads import algo_seed, make_batch, signal_seed  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--log2n", type=int, default=27)
ap.add_argument("--k", type=int, default=10000)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--no-stages", action="store_true",
                help="time the production path (no per-stage events: encode/decode overlapped)")
ap.add_argument("--shards", type=int, default=0,
                help="also run the index-range-sharded split path with G ranks, one "
                     "after another on this GPU, and compare it with the single-GPU result")
a = ap.parse_args()
n, k, delta = 1 << a.log2n, a.k, 1e-6
dev = torch.device("cuda", 0)
sseed = signal_seed(0xC5C50000, 0)
x, truth = make_batch(n, k, [sseed], 20.0, dev, "complex128", magnitude="loguniform_0.1_10",
                      chunk=1)
seeds = np.array([algo_seed(sseed)], dtype=np.uint64)
t0 = time.time()
plan = M.Plan(n, k, M.MultiscaleConfig(), delta, "complex128", 0)
plan_s = time.time() - t0
st = plan.stats()
out = (torch.empty((1, k), dtype=torch.int64, device=dev),
       torch.empty((1, k), dtype=torch.complex128, device=dev),
       torch.empty((1,), dtype=torch.int64, device=dev))
sh = torch.cuda.current_stream().cuda_stream
plan.execute(x, seeds, out=out, stream=sh)  # validating call
if os.environ.get("MSFFT_PROFILE_AFTER_PLAN"):
    torch.cuda.synchronize()
    torch.cuda.profiler.start()  # ncu --profile-from-start off: skip window design
times, stages = [], []
for _ in range(a.reps):
    _, _, _, ms = plan.execute(x, seeds, out=out, assume_valid=True, stream=sh,
                               stage_times=not a.no_stages)
    times.append(ms)
    stages.append(plan.stage_times())
f1, c1, n1 = [t.cpu().numpy() for t in out]
plan.execute(x * 2, seeds, out=out, assume_valid=True, stream=sh)
f2, c2, n2 = [t.cpu().numpy() for t in out]
m = int(n1[0])
shard = None
if a.shards:
    from paper_2011_05698_b200.dist import index_range
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    enc_ms, y = [], None
    for r in range(a.shards):
        lo, hi = index_range(n, r, a.shards)
        xl = x[:, lo:hi].contiguous()
        plan.encode_values(xl, seeds, lo, assume_valid=True)  # warm
        ev[0].record()
        part = plan.encode_values(xl, seeds, lo, assume_valid=True)
        ev[1].record()
        torch.cuda.synchronize()
        enc_ms.append(ev[0].elapsed_time(ev[1]))
        y = part if y is None else y + part
        del xl
    ev[0].record()
    fs, cs, ns = plan.decode_values(y, seeds)
    ev[1].record()
    torch.cuda.synchronize()
    ms_ = int(ns[0])
    index_decode_ms = ev[0].elapsed_time(ev[1])
    fs, cs = fs.cpu().numpy(), cs.cpu().numpy()
    same = bool(ms_ == m and np.array_equal(fs[0, :m], f1[0, :m]))
    rel = float(np.max(np.abs(cs[0, :m] - c1[0, :m]) / np.maximum(np.abs(c1[0, :m]), 1e-300))) \
        if same and m else None
    # tap-range split (x replicated): each part walks 1/G of the taps
    tenc_ms, yt = [], None
    for r in range(a.shards):
        plan.encode_values_part(x, seeds, r, a.shards, assume_valid=True)  # warm
        ev[0].record()
        part = plan.encode_values_part(x, seeds, r, a.shards, assume_valid=True)
        ev[1].record()
        torch.cuda.synchronize()
        tenc_ms.append(ev[0].elapsed_time(ev[1]))
        yt = part if yt is None else yt + part
    ev[0].record()
    ft, ct, nt = plan.decode_values(yt, seeds, folds=True)
    ev[1].record()
    torch.cuda.synchronize()
    dec_folds_ms = ev[0].elapsed_time(ev[1])
    mt = int(nt[0].item())
    ft, ct = ft.cpu().numpy(), ct.cpu().numpy()
    same_t = bool(mt == m and np.array_equal(ft[0, :mt], f1[0, :m]))
    rel_t = float(np.max(np.abs(ct[0, :mt] - c1[0, :m]) / np.maximum(np.abs(c1[0, :m]), 1e-300))) \
        if same_t and m else None
    one = []
    for _ in range(3):
        ev[0].record()
        plan.encode_values_part(x, seeds, 0, 1, assume_valid=True)
        ev[1].record()
        torch.cuda.synchronize()
        one.append(ev[0].elapsed_time(ev[1]))
    shard = {"shards": a.shards, "encode_ms_per_rank": enc_ms,
             "tap_split": {"encode_ms_per_rank": tenc_ms, "encode_ms_one_part": min(one),
                           "bucket_ffts_plus_decode_ms": dec_folds_ms,
                           "same_support_as_single_gpu": same_t,
                           "max_rel_diff_vs_single_gpu": rel_t},
             "bucket_values_mb": y.numel() * 16 / 1e6,
             "decode_ms": index_decode_ms, "same_support_as_single_gpu": same,
             "max_rel_diff_vs_single_gpu": rel}
pos, coef = truth[0]
hit = len(set(f1[0, :m].tolist()) & set(pos.tolist()))
print(json.dumps({
    "config": f"C5: N=2^{a.log2n}, K={k}, complex128, log-uniform |c|, 20 dB",
    "plan_seconds": plan_s, "iterations": st.iterations, "b_first": st.b_first,
    "stage_counts": st.stage_counts, "samples_round_sum": st.samples_round_sum,
    "device_ms": times, "stage_ms_encode_fft_decode": stages[-1],
    "entries": m, "sorted_distinct": bool(np.all(np.diff(f1[0, :m]) > 0)),
    "exact_doubling": bool(np.array_equal(f1, f2) and np.array_equal(c2[0, :m], 2 * c1[0, :m])),
    "true_tones_in_support": hit,
    "sharded": shard,
}))
