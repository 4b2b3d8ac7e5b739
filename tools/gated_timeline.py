"""Timeline of one small-batch gated transform (diagnostic build):

    python tools/build_variant.py tl -DMSFFT_TIMELINE
    MSFFT_B200_LIB=tools/variants/lib_tl.so python tools/gated_timeline.py

For C1, C4 (one signal) and C2 (l=4, q=2): sigma kernel, the encode tasks of
every iteration (first start / last end) and the decode CTA (start, the time
each iteration's gate opened, end), in microseconds from the sigma kernel's
start (%globaltimer), plus the host-measured event time of the call."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_05698_b200 as M  # noqa: E402
from paper_2011_05698_b200 import _lib  # noqa: E402
from paper_2011_05698_b200.workloads import make_signal_np  # noqa: E402

L = _lib.lib()
for name, n, k, l, q, delta, dtype, snr in (("C1", 1 << 16, 50, 16, 1.0, 1e-8, "complex128", None),
                                             ("C4one", 1 << 22, 64, 16, 1.0, 1e-6, "complex64", 25.0),
                                             ("C2_4_2", 1 << 20, 100, 4, 2.0, 1e-6, "complex128", 20.0)):
    x = make_signal_np(n, k, 3, snr, dtype)[0].astype(dtype)
    plan = M.Plan(n, k, M.MultiscaleConfig(l, q), delta, dtype)
    plan.execute(x[None, :], [7])
    ms = []
    for _ in range(5):
        ms.append(plan.execute(x[None, :], [7], assume_valid=True)[3])
    sig = np.zeros(2, np.uint64)
    enc = np.zeros((8192, 6), np.uint64)
    dec = np.zeros((64, 32), np.uint64)
    assert L.msfft_debug_sigma_timeline(sig.ctypes.data_as(C.c_void_p)) == 0
    assert L.msfft_debug_enc_timeline(enc.ctypes.data_as(C.c_void_p), C.c_longlong(8192)) == 0
    assert L.msfft_debug_dec_timeline(dec.ctypes.data_as(C.c_void_p), C.c_longlong(64)) == 0
    t0 = int(enc[enc[:, 1] > 0][:, 0].min())  # the sigma plan is reused: first encode start
    us = lambda t: (int(t) - t0) / 1000.0  # noqa: E731
    used = enc[:, 1] > 0
    e = enc[used]
    e = e[e[:, 0] >= sig[0]]  # this call's tasks
    print(f"== {name}: event ms {np.median(ms):.4f}; sigma {us(sig[0]):.1f}..{us(sig[1]):.1f} us; "
          f"{len(e)} encode tasks")
    for m in sorted(set(e[:, 2].tolist())):
        em = e[e[:, 2] == m]
        print(f"   encode m={m}: {len(em):3d} tasks, start {us(em[:, 0].min()):7.1f}..{us(em[:, 0].max()):7.1f}"
              f", end {us(em[:, 1].min()):7.1f}..{us(em[:, 1].max()):7.1f}")
    for row in e:
        print(f"     task m={int(row[2])}: start {us(row[0]):7.1f} taps {us(row[3]):7.1f} "
              f"gather {us(row[4]):7.1f} end {us(row[1]):7.1f}")
    bt = np.zeros((64, 64), np.int64)
    nb = np.zeros(64, np.int32)
    assert L.msfft_debug_enc_batches(bt.ctypes.data_as(C.c_void_p), nb.ctypes.data_as(C.c_void_p)) == 0
    for i in range(min(4, len(e))):
        k_ = min(int(nb[i]), 64)
        print(f"     cta {i} batches {int(nb[i])}: cycles between batch starts",
              np.diff(bt[i, :k_]).tolist())
    d = dec[0]
    gates = [us(v) for v in d[1:31] if v > 0 and v >= sig[0]]
    print(f"   decode: start {us(d[0]):.1f}, gates " + " ".join(f"{g:.1f}" for g in gates) +
          f", end {us(d[31]):.1f}")
