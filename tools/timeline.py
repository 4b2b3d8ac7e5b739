"""Per-item timeline of the fused C4 launch (diagnostic build):

    python tools/build_variant.py timeline -DMSFFT_TIMELINE
    MSFFT_B200_LIB=tools/variants/lib_timeline.so python tools/timeline.py out.npz

Records {start, end, sm, iteration, code} of every work item of one fused
launch (code >= 0: encode task, < 0: decode of signal -code-1) and prints
the utilisation profile: how many CTA slots hold encode / decode work over
time, and the tail after the last encode item ends."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_05698_b200 as M  # noqa: E402
from paper_2011_05698_b200 import _lib  # noqa: E402
from paper_2011_05698_b200.workloads import algo_seed, make_batch, signal_seed  # noqa: E402

B, n, k = 1024, 1 << 22, 64
dev = torch.device("cuda", 0)
seeds = [signal_seed(0xC4C40000, i) for i in range(B)]
a = np.array([algo_seed(s) for s in seeds], dtype=np.uint64)
x, _ = make_batch(n, k, seeds, 25.0, dev, "complex64")
plan = M.Plan(n, k, M.MultiscaleConfig(), 1e-6, "complex64", 0)
out = (torch.empty((B, k), dtype=torch.int64, device=dev),
       torch.empty((B, k), dtype=torch.complex128, device=dev),
       torch.empty((B,), dtype=torch.int64, device=dev))
plan.execute(x, a, out=out)
for _ in range(3):
    plan.execute(x, a, out=out, assume_valid=True)
torch.cuda.synchronize()
L = _lib.lib()
buf = np.zeros((1 << 16, 3), dtype=np.uint64)
rc = L.msfft_debug_timeline(buf.ctypes.data_as(C.c_void_p), C.c_longlong(1 << 16))
assert rc == 0, rc
used = buf[:, 1] > 0
buf = buf[used]
t0 = buf[:, 0].min()
st = (buf[:, 0] - t0).astype(np.float64) / 1e3
en = (buf[:, 1] - t0).astype(np.float64) / 1e3
sm = (buf[:, 2] >> np.uint64(48)).astype(np.int64)
m = ((buf[:, 2] >> np.uint64(40)) & np.uint64(0xff)).astype(np.int64)
code = (buf[:, 2] & np.uint64(0xffffffff)).astype(np.uint32).view(np.int32).astype(np.int64)
enc = code >= 0
if len(sys.argv) > 1:
    np.savez(sys.argv[1], st=st, en=en, sm=sm, m=m, code=code)
T = en.max()
print(f"items {len(st)} (encode {enc.sum()}, decode {(~enc).sum()}), span {T:.1f} us")
print(f"last encode end {en[enc].max():.1f} us; tail after it {T - en[enc].max():.1f} us")
for mm in sorted(set(m[enc])):
    d = en[enc & (m == mm)] - st[enc & (m == mm)]
    print(f"  encode m={mm}: {d.size} items, mean {d.mean():.1f} us, max {d.max():.1f}")
dd = en[~enc] - st[~enc]
print(f"  decode: mean {dd.mean():.1f} us, p50 {np.median(dd):.1f}, max {dd.max():.1f}")
grid = np.arange(0, T + 10, 10.0)
for g in grid[::10]:
    ae = np.sum(enc & (st <= g) & (en > g))
    ad = np.sum(~enc & (st <= g) & (en > g))
    print(f"  t={g:7.1f} us: encode slots {ae:4d}, decode slots {ad:4d}")
busy = np.sum(en - st)
print(f"slot utilisation {busy / (T * 296):.3f}")
