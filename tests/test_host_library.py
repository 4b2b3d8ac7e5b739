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
