"""Times the 8(f) signal helpers on the GPU against the reference's own CPU
code (oracle/_ref) at the C4 signal size (N=2^22, K=64), and prints one JSON
line (kept under profiles/).  GPU times: CUDA-event/wall time of the C-ABI
call with device-resident buffers, after a warm-up call; CPU: one call."""
import json
import os
import sys
import tempfile
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_05698_b200.signal as S  # noqa: E402
from oracle import available, load  # noqa: E402

n, k = 1 << int(os.environ.get("LOG2N", "22")), 64
R = load("reference" if available("reference") else "port")
dev = torch.device("cuda", 0)
res = {"n": n, "k": k, "cpu_kind": R.kind}


def gpu_time(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3, out


def cpu_time(fn):
    t0 = time.perf_counter()
    out = fn()
    return (time.perf_counter() - t0) * 1e3, out


g_ms, (x, f, c, exact) = gpu_time(lambda: S.generate_test_signal(n, k, 77, "complex128", dev))
c_ms, (rx, rf, rc) = cpu_time(lambda: R.generate_test_signal(n, k, 77))
res["generate_test_signal"] = {"gpu_ms": g_ms, "cpu_ms": c_ms, "bit_exact": bool(
    exact and np.array_equal(x.cpu().numpy(), rx))}
g_ms, y = gpu_time(lambda: S.add_awgn(x, 20.0, 5))
c_ms, _ = cpu_time(lambda: R.add_awgn(rx, 20.0, 5))
res["add_awgn"] = {"gpu_ms": g_ms, "cpu_ms": c_ms}
g_ms, X = gpu_time(lambda: S.dft_dense(y))
yh = y.cpu().numpy()
c_ms, RX = cpu_time(lambda: R.dft_dense(yh))
res["dft_dense"] = {"gpu_ms": g_ms, "cpu_ms": c_ms,
                    "bit_exact": bool(np.array_equal(X.cpu().numpy(), RX))}
g_ms, (tf, tc) = gpu_time(lambda: S.top_k_spectrum(X, k))
c_ms, (qf, qc) = cpu_time(lambda: R.top_k_spectrum(RX, k))
res["top_k_spectrum"] = {"gpu_ms": g_ms, "cpu_ms": c_ms,
                         "identical": bool(np.array_equal(tf, qf) and np.array_equal(tc, qc))}
d = tempfile.mkdtemp()
g_ms, _ = gpu_time(lambda: S.write_signal_file(os.path.join(d, "a.msft"), y), reps=2)
c_ms, _ = cpu_time(lambda: R.write_signal_file(os.path.join(d, "b.msft"), yh))
res["write_signal_file"] = {"gpu_ms": g_ms, "cpu_ms": c_ms, "bytes": 16 + 16 * n}
g_ms, z = gpu_time(lambda: S.read_signal_file(os.path.join(d, "b.msft"), "complex128", dev), reps=2)
c_ms, _ = cpu_time(lambda: R.read_signal_file(os.path.join(d, "a.msft"), n))
res["read_signal_file"] = {"gpu_ms": g_ms, "cpu_ms": c_ms,
                           "identical": bool(np.array_equal(z.cpu().numpy(), yh))}
print(json.dumps(res))
