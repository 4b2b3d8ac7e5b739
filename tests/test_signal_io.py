"""SURVEY 8(f) rows 2-3 on the host: MSFT signal files, truth CSV and
error_metrics through the C ABI, against the reference's own io.cpp /
signal.cpp (oracle) -- byte-identical files, identical metrics, the same
exception types and messages.  No GPU needed (host buffers)."""
import os

import numpy as np
import pytest

import paper_2011_05698_b200 as M
import paper_2011_05698_b200.signal as S
from conftest import oracle_kinds


@pytest.fixture(scope="module", params=oracle_kinds())
def orc(request):
    from oracle import load
    return load(request.param)


def _sig(orc, n=4096, k=20, seed=5):
    x, f, c = orc.generate_test_signal(n, k, seed)
    return x, f, c


def test_signal_file_bytes_identical(orc, tmp_path):
    x, _, _ = _sig(orc)
    S.write_signal_file(tmp_path / "a.msft", x)
    orc.write_signal_file(tmp_path / "b.msft", x)
    a = (tmp_path / "a.msft").read_bytes()
    assert a == (tmp_path / "b.msft").read_bytes()
    assert a[:8] == b"MSFT\0\0\0\0" and int.from_bytes(a[8:16], "little") == 4096
    assert np.array_equal(S.read_signal_file(tmp_path / "b.msft"), x)
    assert np.array_equal(orc.read_signal_file(tmp_path / "a.msft"), x)
    assert S.signal_file_length(tmp_path / "a.msft") == 4096


def test_signal_file_complex64(tmp_path):
    x = (np.arange(64) * (1 + 0.5j)).astype(np.complex64)
    S.write_signal_file(tmp_path / "a.msft", x)  # exact upcast to float64 pairs
    back = S.read_signal_file(tmp_path / "a.msft")
    assert back.dtype == np.complex128 and np.array_equal(back, x.astype(np.complex128))
    assert np.array_equal(S.read_signal_file(tmp_path / "a.msft", "complex64"), x)


@pytest.mark.parametrize("blob,msg", [
    (b"XXXX\0\0\0\0" + (64).to_bytes(8, "little"), "bad magic"),
    (b"MSF", "bad magic"),
    (b"MSFT\0\0\0\0" + (48).to_bytes(8, "little"), "bad length field"),
    (b"MSFT\0\0\0\0" + (2).to_bytes(8, "little"), "bad length field"),
    (b"MSFT\0\0\0\0" + (1 << 31).to_bytes(8, "little"), "bad length field"),
    (b"MSFT\0\0\0\0" + (64).to_bytes(8, "little") + b"\0" * 100, "truncated file"),
])
def test_signal_file_errors_match_reference(orc, tmp_path, blob, msg):
    p = tmp_path / "bad.msft"
    p.write_bytes(blob)
    with pytest.raises(RuntimeError, match=msg) as ours:
        S.read_signal_file(p)
    with pytest.raises(Exception) as ref:
        orc.read_signal_file(p)
    assert str(ours.value) == str(ref.value)


def test_signal_file_validation(orc, tmp_path):
    x = np.zeros(64, np.complex128)
    x[7] = np.nan
    with pytest.raises(M.InvalidArgument, match="ComplexSignal: non-finite sample"):
        S.write_signal_file(tmp_path / "a.msft", x)
    assert not (tmp_path / "a.msft").exists()
    with pytest.raises(M.InvalidArgument, match="ComplexSignal: n must be a power of two >= 4"):
        S.write_signal_file(tmp_path / "a.msft", np.zeros(48, np.complex128))
    # a file holding a NaN: read validates (io.cpp:52)
    blob = b"MSFT\0\0\0\0" + (4).to_bytes(8, "little") + np.array(
        [0, 0, np.inf, 0, 0, 0, 0, 0], "<f8").tobytes()
    (tmp_path / "nan.msft").write_bytes(blob)
    with pytest.raises(M.InvalidArgument, match="ComplexSignal: non-finite sample"):
        S.read_signal_file(tmp_path / "nan.msft")
    with pytest.raises(Exception, match="ComplexSignal: non-finite sample"):
        orc.read_signal_file(tmp_path / "nan.msft")
    with pytest.raises(RuntimeError, match="read_signal_file: cannot open"):
        S.read_signal_file(tmp_path / "missing.msft")
    with pytest.raises(RuntimeError, match="write_signal_file: cannot open"):
        S.write_signal_file(tmp_path / "no" / "dir.msft", np.zeros(4, np.complex128))


def test_truth_csv_bytes_identical(orc, tmp_path):
    _, f, c = _sig(orc, 8192, 50, 11)
    S.write_truth_csv(tmp_path / "a.csv", f, c)
    orc.write_truth_csv(tmp_path / "b.csv", 8192, f, c)
    assert (tmp_path / "a.csv").read_text() == (tmp_path / "b.csv").read_text()
    f2, c2 = S.read_truth_csv(tmp_path / "b.csv", 8192)
    assert np.array_equal(f2, f) and np.array_equal(c2, c)
    # unsorted input with a duplicate: std::map order, the last value wins
    S.write_truth_csv(tmp_path / "u.csv", [9, 3, 9], [1, 2, 3 + 1j])
    assert (tmp_path / "u.csv").read_text() == "position,re,im\n3,2,0\n9,3,1\n"


def test_truth_csv_validation(orc, tmp_path):
    p = tmp_path / "t.csv"
    p.write_text("position,re,im\n5,1,0\n70,0,1\n")
    with pytest.raises(M.InvalidArgument, match="SparseSpectrum: position out of range"):
        S.read_truth_csv(p, 64)
    with pytest.raises(Exception, match="SparseSpectrum: position out of range"):
        orc.read_truth_csv(p, 64)
    p.write_text("position,re,im\n5,nan,0\n")
    with pytest.raises(M.InvalidArgument, match="SparseSpectrum: non-finite coefficient"):
        S.read_truth_csv(p, 64)
    with pytest.raises(M.InvalidArgument, match="SparseSpectrum: n must be a power of two"):
        S.read_truth_csv(p, 48)
    p.write_text("position,re,im\n\n7,0.5,-0.25\n")
    f, c = S.read_truth_csv(p, 64)
    assert list(f) == [7] and c[0] == 0.5 - 0.25j


def test_error_metrics_match_reference(orc):
    rng = np.random.default_rng(3)
    _, f, c = _sig(orc, 8192, 50, 4)
    cases = [
        (f, c, 50),                                  # exact: all zero
        (f[1:], c[1:], 50),                          # one missing unit tone: l1 = 0.02
        (np.r_[f, [int(np.setdiff1d(np.arange(8192), f)[0])]], np.r_[c, [1]], 50),  # spurious
        (f, c * (1 + 1e-7), 50),                     # all below the l0 threshold
        (f[::2], c[::2] + rng.normal(size=25), 50),
        (f, c, 7),
    ]
    for ef, ec, k in cases:
        m = S.error_metrics(8192, f, c, 8192, ef, ec, k)
        assert (m.l0_err, m.l1_err, m.l2_err) == orc.error_metrics(8192, f, c, ef, ec, k)
    m = S.error_metrics(8192, f, c, 8192, f[1:], c[1:], 50)
    assert m.l0_err == 1 and abs(m.l1_err - 0.02) < 1e-15
    assert S.error_metrics(8192, f, c, 8192, f, c, 50) == S.EvalMetrics(0, 0.0, 0.0)
    assert S.error_metrics(64, [], [], 64, [], [], 0) == S.EvalMetrics()
    with pytest.raises(M.InvalidArgument, match="error_metrics: k = 0 with nonempty support union"):
        S.error_metrics(64, [3], [1], 64, [], [], 0)
    with pytest.raises(M.InvalidArgument, match="error_metrics: size mismatch"):
        S.error_metrics(64, [3], [1], 128, [3], [1], 1)


def test_port_signal_helpers_match_reference(tmp_path):
    """The restatement (oracle/port) agrees with the reference bit-for-bit on
    the 8(f) helpers (it stands in for the reference where that is absent)."""
    from oracle import available, load
    if not (available("reference") and available("port")):
        pytest.skip("needs both oracles")
    R, P = load("reference"), load("port")
    rng = np.random.default_rng(1)
    for n in (64, 4096, 1 << 15):
        x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        a = R.dft_dense(x)
        assert np.array_equal(a, P.dft_dense(x))
        assert np.array_equal(R.idft_dense(a), P.idft_dense(a))
        fr, cr = R.top_k_spectrum(a, 17)
        fp, cp = P.top_k_spectrum(a, 17)
        assert np.array_equal(fr, fp) and np.array_equal(cr, cp)
    x, f, c = R.generate_test_signal(8192, 50, 21)
    assert np.array_equal(P.synthesize(8192, f, c), x)
    assert np.array_equal(R.synthesize(8192, f, c), x)
