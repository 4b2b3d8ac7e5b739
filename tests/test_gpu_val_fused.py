"""The validating fused launch (fused.cu fused_val_kernel): one persistent
kernel that runs ComplexSignal::validate's scan (proj/src/signal.cpp:22-25,
called on every sfft4 entry, proj/src/sfft4.cpp:133), the encode (as packed
per-signal items) and the decode.  It must give bit-for-bit the outputs of
the separate scan + fused kernel, reject a non-finite sample anywhere with the
reference's message, and leave its counters clean for the next call."""
import ctypes as C

import numpy as np
import pytest

import paper_2011_05698_b200 as M
from paper_2011_05698_b200 import _lib as L

pytestmark = pytest.mark.gpu


def _signals(n, batch, dtype, seed):
    rng = np.random.default_rng(seed)
    x = np.zeros((batch, n), np.complex128)
    for s in range(batch):
        spec = np.zeros(n, np.complex128)
        pos = rng.choice(n, 40, replace=False)
        spec[pos] = np.exp(2j * np.pi * rng.random(40))
        x[s] = np.fft.ifft(spec) * n
    x += 0.01 * (rng.standard_normal(x.shape) + 1j * rng.standard_normal(x.shape))
    return x.astype(dtype)


def _plan(monkeypatch, n, k, dtype, **env):
    for key in ("MSFFT_VAL_FUSED", "MSFFT_VAL_CHUNK_MB", "MSFFT_VAL_ITEM_KB", "MSFFT_VAL_DLAG",
                "MSFFT_VAL_ELAG"):
        monkeypatch.delenv(key, raising=False)
    for key, v in env.items():
        monkeypatch.setenv(key, str(v))
    return M.Plan(n, k, M.MultiscaleConfig(), 1e-6, dtype)


@pytest.mark.parametrize("dtype", ["complex64", "complex128"])
@pytest.mark.parametrize("env", [
    {},                                                   # one chunk
    {"MSFFT_VAL_CHUNK_MB": 1, "MSFFT_VAL_ITEM_KB": 48},   # many chunks, ragged items
    {"MSFFT_VAL_CHUNK_MB": 1, "MSFFT_VAL_DLAG": 0, "MSFFT_VAL_ELAG": 2},
])
def test_val_fused_bit_identical(monkeypatch, dtype, env):
    import torch
    n, k, batch = 1 << 16, 50, 37
    x = torch.as_tensor(_signals(n, batch, np.dtype(dtype), 5)).cuda()
    seeds = np.arange(100, 100 + batch, dtype=np.uint64)
    pv = _plan(monkeypatch, n, k, dtype, **env)
    assert pv.launches(batch) == 2  # sigma + the validating fused launch
    fv, cv, nv, _ = pv.execute(x, seeds)
    pr = _plan(monkeypatch, n, k, dtype, MSFFT_VAL_FUSED=0)
    assert pr.launches(batch) == 3  # sigma + scan + fused
    fr, cr, nr, _ = pr.execute(x, seeds)
    fa, ca, na, _ = pr.execute(x, seeds, assume_valid=True)
    assert np.array_equal(nv, nr) and np.array_equal(fv, fr) and np.array_equal(cv, cr)
    assert np.array_equal(nv, na) and np.array_equal(fv, fa) and np.array_equal(cv, ca)
    assert (nv > 0).all()
    # repeated calls reuse the counters the last CTA reset
    fv2, cv2, nv2, _ = pv.execute(x, seeds)
    assert np.array_equal(fv2, fv) and np.array_equal(cv2, cv)


@pytest.mark.parametrize("dtype", ["complex64", "complex128"])
def test_val_fused_rejects_non_finite(monkeypatch, dtype):
    import torch
    n, k, batch = 1 << 16, 50, 24
    xs = _signals(n, batch, np.dtype(dtype), 9)
    seeds = np.arange(batch, dtype=np.uint64)
    pv = _plan(monkeypatch, n, k, dtype, MSFFT_VAL_CHUNK_MB=1, MSFFT_VAL_ITEM_KB=48)
    good = pv.execute(torch.as_tensor(xs).cuda(), seeds)
    rng = np.random.default_rng(3)
    cases = [(0, 0), (batch - 1, n - 1), (batch // 2, n // 2), (5, 6143), (5, 6144),
             (int(rng.integers(batch)), int(rng.integers(n)))]
    for (s, i), bad in zip(cases, [np.nan, np.inf, -np.inf, np.nan, np.inf, np.nan]):
        for part in ("re", "im"):
            y = xs.copy()
            y[s, i] = complex(bad, 0.0) if part == "re" else complex(0.0, bad)
            with pytest.raises(M.InvalidArgument, match="ComplexSignal: non-finite sample"):
                pv.execute(torch.as_tensor(y).cuda(), seeds)
    # the plan is clean after the failures
    again = pv.execute(torch.as_tensor(xs).cuda(), seeds)
    for a, b in zip(good[:3], again[:3]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("dtype", ["complex64", "complex128"])
def test_val_fused_strided_rows(monkeypatch, dtype):
    """Rows of a wider buffer through the C ABI (x_stride > n): the padding
    (NaN) is never read, the rows give the contiguous batch's outputs."""
    import torch
    n, k, batch, pad = 1 << 16, 50, 20, 16
    xs = _signals(n, batch, np.dtype(dtype), 13)
    seeds = np.arange(7, 7 + batch, dtype=np.uint64)
    pv = _plan(monkeypatch, n, k, dtype, MSFFT_VAL_CHUNK_MB=2)
    ref = pv.execute(torch.as_tensor(xs).cuda(), seeds)
    wide = np.full((batch, n + pad), np.nan, xs.dtype)
    wide[:, :n] = xs
    t = torch.as_tensor(wide).cuda()
    f = np.zeros((batch, k), np.int64)
    c = np.zeros((batch, k), np.complex128)
    cnt = np.zeros(batch, np.int64)
    err = C.create_string_buffer(1024)
    ms = C.c_double()
    st = pv._lib.msfft_execute(pv._h, batch, C.c_void_p(t.data_ptr()), n + pad, L.MSFFT_DEVICE,
                               seeds.ctypes.data_as(C.POINTER(C.c_uint64)),
                               C.c_void_p(f.ctypes.data), C.c_void_p(c.ctypes.data),
                               C.c_void_p(cnt.ctypes.data), L.MSFFT_HOST, 0, None, C.byref(ms),
                               err, 1024)
    assert st == 0, err.value
    assert np.array_equal(cnt, ref[2]) and np.array_equal(f, ref[0]) and np.array_equal(c, ref[1])
