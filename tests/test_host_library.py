"""The C-ABI library on a machine without a GPU: it loads, exports every
symbol include/msfft_b200.h declares, computes the host-side plan pieces
exactly like the reference, and refuses to compute without a device (there
is no CPU fallback).  CPU only."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import REPO


@pytest.fixture(scope="session")
def lib():
    from paper_2011_05698_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2011_05698_b200.build import build
        build()
    return _lib.lib()


def header_functions():
    text = open(os.path.join(REPO, "include", "msfft_b200.h")).read()
    return sorted(set(re.findall(r"^[A-Za-z_][\w \*]*?\b(msfft_\w+)\(", text, re.M)))


def test_exports_every_declared_symbol(lib):
    from paper_2011_05698_b200 import _lib
    names = header_functions()
    assert len(names) >= 14
    for name in names:
        assert hasattr(lib, name), f"{name} declared in msfft_b200.h but not exported"
    assert set(names) == set(_lib.EXPORTED)


def test_version(lib):
    assert b"sm_100a" in lib.msfft_version()


def test_sigma_plan_matches_reference(lib, golden):
    g = golden("known_answers")
    for key in ("random_params", "random_params_big"):
        rp = g[key]
        m = len(rp["sigma"])
        s = np.zeros(m, np.int64)
        si = np.zeros(m, np.int64)
        err = C.create_string_buffer(256)
        st = lib.msfft_sigma_plan(rp["seed"], rp["n"], m, s.ctypes.data_as(C.POINTER(C.c_int64)),
                                  si.ctypes.data_as(C.POINTER(C.c_int64)), err, 256)
        assert st == 0, err.value
        assert list(s) == rp["sigma"] and list(si) == rp["sigma_inv"]


def test_tau_plan_matches_reference(lib, oracle):
    for n in (1 << 16, 1 << 22):
        for b in (32, 256, 4096):
            for l, q in ((16, 1.0), (8, 2.0), (4, 1.0), (8, 4.0), (2, 0.0)):
                L = n // b
                taus = np.zeros(64, np.int64)
                rounds = C.c_int32()
                err = C.create_string_buffer(256)
                st = lib.msfft_tau_plan(float(L), n, l, q, taus.ctypes.data_as(C.POINTER(C.c_int64)),
                                        64, C.byref(rounds), err, 256)
                assert st == 0, err.value
                stages = oracle.stage_count(L, l, q)
                assert rounds.value == stages + 1
                want, ln = [0], float(L)
                for _ in range(stages):
                    want.append(oracle.tau_schedule(ln, n))
                    ln *= (q + 1.0) / l
                assert list(taus[: rounds.value]) == want


def test_tau_plan_rejects_bad_config(lib):
    taus = np.zeros(8, np.int64)
    rounds = C.c_int32()
    err = C.create_string_buffer(256)
    st = lib.msfft_tau_plan(32.0, 1024, 2, 1.0, taus.ctypes.data_as(C.POINTER(C.c_int64)), 8,
                            C.byref(rounds), err, 256)
    assert st == 1 and err.value == b"MultiscaleConfig: l/(q+1) must exceed 1"


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # noqa: BLE001
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-device behaviour")
def test_no_cpu_fallback(lib):
    import paper_2011_05698_b200 as M
    x = np.zeros(1 << 12, np.complex128)
    with pytest.raises(M.CudaError):
        M.sfft4(x, 10)
    with pytest.raises(M.CudaError):
        M.Plan(1 << 12, 10)
    assert lib.msfft_device_count() == 0


def test_host_plan_helpers_match_reference(lib, golden):
    """The reference's scalar plan helpers through the C ABI (host code, no
    device): mod_inverse, bucket_of, stage_count, tau_schedule,
    check_parameter_bounds, MultiscaleConfig::validate -- against the
    known answers generated from the reference."""
    import paper_2011_05698_b200 as M
    from paper_2011_05698_b200 import components as CMP
    ka = golden("known_answers")
    for L, l, q, want in ka["stage_count"]:
        assert CMP.stage_count(L, M.MultiscaleConfig(l, q)) == want
    for ln, n, want in ka["tau_schedule"]:
        assert CMP.tau_schedule(ln, n) == want
    for s, n, want in ka["mod_inverse"]:
        assert CMP.mod_inverse(s, n) == want
    for u, L, b, want in ka["bucket_of"]:
        assert CMP.bucket_of(u, L, b) == want
    ok, qm = CMP.check_parameter_bounds(0.3, 4)
    assert ok and qm.hex() == ka["check_parameter_bounds"][0][3]
    with pytest.raises(M.InvalidArgument, match="mod_inverse: sigma must be odd"):
        CMP.mod_inverse(4, 16)
    with pytest.raises(M.InvalidArgument, match="mod_inverse: n must be a power of two"):
        CMP.mod_inverse(3, 12)
    with pytest.raises(M.InvalidArgument, match="max_dphi must be positive"):
        CMP.check_parameter_bounds(0.0, 4)
    # the reference would loop forever here; the drop-in reports the config error
    with pytest.raises(M.InvalidArgument, match="l/\\(q\\+1\\) must exceed 1"):
        CMP.stage_count(32, M.MultiscaleConfig(2, 1.0))
    err = C.create_string_buffer(256)
    assert lib.msfft_config_validate(1, 1.0, err, 256) == 1
    assert err.value == b"MultiscaleConfig: l must be >= 2"
    assert lib.msfft_config_validate(16, -1.0, err, 256) == 1
    assert err.value == b"MultiscaleConfig: q must be >= 0"
    assert lib.msfft_config_validate(16, 1.0, err, 256) == 0
    assert lib.msfft_bucket_of(5, 0, 32) == -1


def test_validate_signal_host_order(lib):
    """ComplexSignal::validate on host memory needs no device: the reference's
    check order and messages (signal.cpp:18-26)."""
    import paper_2011_05698_b200 as M
    with pytest.raises(M.InvalidArgument, match="n must be a power of two >= 4"):
        M.validate_signal(np.full(6, np.nan, np.complex128))
    with pytest.raises(M.InvalidArgument, match="sample count != n"):
        M.validate_signal(np.full(8, np.nan, np.complex64), n=16)
    x = np.zeros((3, 16), np.complex64)
    assert M.validate_signal(x) == 0.0
    x[2, 15] = complex(np.inf, 0)
    with pytest.raises(M.InvalidArgument, match="non-finite sample"):
        M.validate_signal(x)


def test_cpp_header_runs_host_helpers_without_device(tmp_path):
    """The drop-in's host-side pieces (Rng, random_params, mod_inverse,
    bucket_of, stage_count, tau_schedule, initial_region, SparseSpectrum::
    validate, random_sparse_spectrum) agree with the reference library on a
    machine without a GPU."""
    import shutil
    import subprocess
    if not shutil.which("g++"):
        pytest.skip("g++ not available")
    refdir = os.path.join(REPO, "oracle", "_ref")
    if not os.path.exists(os.path.join(refdir, "libmsfft_ref.so")):
        pytest.skip("reference oracle library not built")
    src = tmp_path / "host.cpp"
    src.write_text(r'''
#define MSFFT_B200_AS_MSFFT
#include <cstdio>
#include "../oracle/oracle_api.h"
#include "msfft_b200.hpp"
int main() {
    int bad = 0;
    msfft::Rng r(12345);
    std::vector<int64_t> s(8), si(8);
    char err[256];
    orc_random_params(1 << 22, 12345, 8, s.data(), si.data(), err, sizeof(err));
    for (int i = 0; i < 8; ++i) {
        auto p = msfft::random_params(1 << 22, r, 0);
        bad += p.sigma != s[i] || p.sigma_inv != si[i] || p.tau != 0;
    }
    for (double len : {2.0, 32.0, 2048.0, 131072.0})
        bad += msfft::stage_count(len, msfft::MultiscaleConfig{16, 1.0}) != orc_stage_count(len, 16, 1.0);
    bad += msfft::tau_schedule(32, 8192) != 256;
    bad += msfft::bucket_of(8192 - 16, 32, 256) != orc_bucket_of(8192 - 16, 32, 256);
    auto reg = msfft::initial_region(3, 64);
    bad += reg.u_min != 160.0 || reg.length != 64.0 || reg.stage != 1;
    msfft::Rng g(77);
    auto spec = msfft::random_sparse_spectrum(8192, 50, g);
    bad += spec.entries.size() != 50;
    spec.validate();
    msfft::Rng a(5), b(5);
    for (int i = 0; i < 100; ++i) bad += a.gaussian() != b.gaussian();
    std::printf("bad=%d\n", bad);
    return bad;
}
''')
    exe = str(tmp_path / "host")
    inc = os.path.join(REPO, "include")
    libdir = os.path.join(REPO, "paper_2011_05698_b200")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", inc, "-I", os.path.join(REPO, "include"),
                    "-include", "cstdint", str(src), "-L", libdir, "-lmsfft_b200", "-L", refdir,
                    "-lmsfft_ref", "-o", exe], check=True, cwd=os.path.join(REPO, "include"))
    env = dict(os.environ, LD_LIBRARY_PATH=f"{libdir}:{refdir}")
    r = subprocess.run([exe], env=env, capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "bad=0" in r.stdout
