"""ComplexSignal::validate (proj/src/signal.cpp:18-26) on the device: the
TMA-staged finiteness scan (engine.cu validate_kernel) against numpy's
isfinite on the same bytes -- every position class of a chunk (first, last,
chunk boundaries, partial last chunk), NaN / +-Inf in either component,
complex64 and complex128, contiguous batches and strided rows."""
import numpy as np
import pytest

import paper_2011_05698_b200 as M

pytestmark = pytest.mark.gpu


def _dev(a):
    import torch
    return torch.as_tensor(a).cuda()


@pytest.mark.parametrize("dtype", [np.complex64, np.complex128])
@pytest.mark.parametrize("n,batch", [(4, 1), (8, 3), (1024, 5), (1 << 13, 2), (1 << 16, 9)])
def test_validate_positions(dtype, n, batch):
    rng = np.random.default_rng(n * 7 + batch)
    x = (rng.standard_normal((batch, n)) + 1j * rng.standard_normal((batch, n))).astype(dtype)
    assert M.validate_signal(_dev(x)) >= 0.0
    flat = x.size
    esz = np.dtype(dtype).itemsize
    chunk = 16384 // esz  # samples per 16-KB chunk
    cand = {0, flat - 1, flat // 2, min(chunk, flat - 1), min(chunk - 1, flat - 1),
            min(2 * chunk + 1, flat - 1), int(rng.integers(0, flat))}
    for pos in sorted(cand):
        for bad in (np.nan, np.inf, -np.inf):
            for part in ("re", "im"):
                y = x.copy().reshape(-1)
                y[pos] = complex(bad, 0.0) if part == "re" else complex(0.0, bad)
                y = y.reshape(batch, n)
                assert not np.isfinite(y).all()
                with pytest.raises(M.InvalidArgument, match="ComplexSignal: non-finite sample"):
                    M.validate_signal(_dev(y))


@pytest.mark.parametrize("dtype", [np.complex64, np.complex128])
def test_validate_strided_rows(dtype):
    """Rows of a wider buffer (x_stride > n): padding is never read."""
    import torch
    n, batch, stride = 1 << 12, 6, (1 << 12) + 8
    base = np.zeros((batch, stride), dtype)
    base[:, n:] = np.nan  # outside the rows
    t = _dev(base)
    fn = M._L.lib().msfft_validate_signal  # the C ABI directly: stride != n
    import ctypes as C
    err = C.create_string_buffer(256)
    out = C.c_double()
    code = M._L.MSFFT_C64 if dtype == np.complex64 else M._L.MSFFT_C128
    st = fn(C.c_void_p(t.data_ptr()), n, n, batch, stride, code, M._L.MSFFT_DEVICE, None,
            C.byref(out), err, 256)
    assert st == 0, err.value
    t[batch - 1, n - 1] = complex(0.0, np.inf)
    st = fn(C.c_void_p(t.data_ptr()), n, n, batch, stride, code, M._L.MSFFT_DEVICE, None,
            C.byref(out), err, 256)
    assert st == M._L.MSFFT_ERR_INVALID_ARGUMENT
    assert err.value.decode() == "ComplexSignal: non-finite sample"
    torch.cuda.synchronize()


def test_validate_order_and_messages():
    with pytest.raises(M.InvalidArgument, match="n must be a power of two >= 4"):
        M.validate_signal(_dev(np.full(6, np.nan, np.complex64)))
    with pytest.raises(M.InvalidArgument, match="sample count != n"):
        M.validate_signal(_dev(np.full(8, np.nan, np.complex64)), n=16)


def test_execute_rejects_non_finite_batch():
    """A validating batched execute raises for a NaN in any signal of the
    batch; ASSUME_VALID skips the scan."""
    import torch
    n, k, batch = 1 << 14, 8, 6
    plan = M.Plan(n, k, M.MultiscaleConfig(), 1e-6, "complex64")
    x = torch.randn((batch, n), dtype=torch.complex64, device="cuda")
    seeds = np.arange(batch, dtype=np.uint64)
    plan.execute(x, seeds)
    x[batch - 1, n - 1] = complex(float("nan"), 0.0)
    with pytest.raises(M.InvalidArgument, match="non-finite sample"):
        plan.execute(x, seeds)
    plan.execute(x, seeds, assume_valid=True)
