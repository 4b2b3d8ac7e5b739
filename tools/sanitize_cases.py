"""Small cases that drive every kernel path once, for the checked build
(compute-sanitizer is closed on the GPU pool):

    python tools/build_variant.py checked -DMSFFT_CHECKED
    MSFFT_B200_LIB=tools/variants/lib_checked.so python tools/sanitize_cases.py [case ...]

Cases (all by default): fused batch, serial encode/decode, one-CTA large-size
decode, wide decode, sparse host ingest, async + PDL chain, window designer,
signal helpers, phase Monte Carlo.  Sizes are small (the whole run takes
seconds) while still reaching the code path named.
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_05698_b200 as M  # noqa: E402
from paper_2011_05698_b200 import signal as S  # noqa: E402
from paper_2011_05698_b200.workloads import make_batch, make_signal_np  # noqa: E402

dev = torch.device("cuda", 0)


def _out(b, k):
    return (torch.empty((b, k), dtype=torch.int64, device=dev),
            torch.empty((b, k), dtype=torch.complex128, device=dev),
            torch.empty((b,), dtype=torch.int64, device=dev))


def _env(**kv):
    for key, v in kv.items():
        if v is None:
            os.environ.pop(key, None)
        else:
            os.environ[key] = str(v)


def case_fused():
    n, k, B = 1 << 16, 20, 24
    x, _ = make_batch(n, k, list(range(B)), 20.0, dev, "complex64")
    plan = M.Plan(n, k, M.MultiscaleConfig(), 1e-6, "complex64")
    o = _out(B, k)
    plan.execute(x, np.arange(B, dtype=np.uint64), out=o)
    assert int(o[2].min()) > 0


def case_serial():
    n, k, B = 1 << 16, 20, 6
    x, _ = make_batch(n, k, list(range(B)), 20.0, dev, "complex128")
    plan = M.Plan(n, k, M.MultiscaleConfig(), 1e-6, "complex128")
    o = _out(B, k)
    plan.execute(x, np.arange(B, dtype=np.uint64), out=o, serial=True)
    assert int(o[2].min()) > 0


def _big_signal():
    x, _, _ = make_signal_np(1 << 18, 3000, 5, None, "complex128", "loguniform_0.1_10")
    return torch.as_tensor(x[None, :]).to(dev)


def case_big_cta():
    _env(MSFFT_WIDE_MAX_BATCH=0)
    plan = M.Plan(1 << 18, 3000, M.MultiscaleConfig(), 1e-8, "complex128")
    o = _out(1, 3000)
    plan.execute(_big_signal(), [123], out=o)
    _env(MSFFT_WIDE_MAX_BATCH=None)
    assert int(o[2][0]) > 0


def case_wide():
    plan = M.Plan(1 << 18, 3000, M.MultiscaleConfig(), 1e-8, "complex128")
    o = _out(1, 3000)
    plan.execute(_big_signal(), [123], out=o)
    assert int(o[2][0]) > 0


def case_ingest():
    _env(MSFFT_INGEST_CHUNK=2, MSFFT_DMA_VALIDATE_SHARE=0.5)
    n, k, B = 1 << 18, 20, 5
    x, _ = make_batch(n, k, list(range(B)), 20.0, dev, "complex64")
    xh = x.cpu().pin_memory()
    plan = M.Plan(n, k, M.MultiscaleConfig(), 1e-6, "complex64")
    assert plan.ingest_samples_per_signal > 0
    f, c, cnt, _ = plan.execute(xh, np.arange(B, dtype=np.uint64))
    f2, c2, cnt2, _ = plan.execute(xh.numpy(), np.arange(B, dtype=np.uint64))
    _env(MSFFT_INGEST_CHUNK=None, MSFFT_DMA_VALIDATE_SHARE=None)
    assert np.array_equal(f, f2) and np.array_equal(cnt, cnt2)


def case_pdl():
    _env(MSFFT_PDL=1)
    n, k, B = 1 << 12, 8, 320
    rng = np.random.default_rng(5)
    xs = (rng.standard_normal((B, n)) + 1j * rng.standard_normal((B, n))).astype(np.complex64)
    xs[:, 0] += 50.0
    xd = torch.as_tensor(xs).to(dev)
    plan = M.Plan(n, k, M.MultiscaleConfig(), 1e-6, "complex64")
    outs = [_out(B, k) for _ in range(3)]
    for i, o in enumerate(outs):
        plan.execute(xd, np.arange(B, dtype=np.uint64) + np.uint64(1000 * (i % 2)), out=o,
                     assume_valid=True, async_=True)
    plan.sync()
    _env(MSFFT_PDL=None)
    assert torch.equal(outs[0][0], outs[2][0])


def case_window():
    w = M.window(1 << 16, 64, 1e-8, device=0)
    assert w is not None


def case_signal():
    x, f, c, _ = S.generate_test_signal(1 << 14, 12, 3, "complex128", dev)
    y = S.add_awgn(x, 20.0, 9)
    spec = S.dft_dense(y[: 1 << 12])
    S.top_k_spectrum(spec, 12)
    S.idft_dense(spec)
    S.synthesize(1 << 12, np.arange(0, 1 << 12, 400), c[:11], "complex64", dev)


def case_phase():
    S.run_phase_experiment(1 << 12, 8, 64, [10.0, 30.0], 64, 11, keep_trials=True)


CASES = {name[5:]: fn for name, fn in globals().items() if name.startswith("case_")}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for name in names:
        t0 = time.time()
        CASES[name]()
        torch.cuda.synchronize()
        print(f"ok {name} ({time.time() - t0:.1f} s)", flush=True)
