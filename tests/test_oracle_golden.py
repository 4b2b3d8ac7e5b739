"""Pins the CPU oracles (the compiled reference and the restatement in
oracle/port) against the golden fixtures generated from the reference
itself (tests/golden/make_golden.py).  CPU only."""
import hashlib

import numpy as np
import pytest

from conftest import oracle_kinds
from helpers import golden_result, make_signal

KINDS = oracle_kinds()
pytestmark = pytest.mark.skipif(not KINDS, reason="no oracle library built")


@pytest.fixture(params=KINDS, scope="module")
def orc(request):
    from oracle import load
    return load(request.param)


def test_known_answers(orc, golden):
    g = golden("known_answers")
    for L, n, tau in g["tau_schedule"]:
        assert orc.tau_schedule(L, n) == tau
    # SPEC.md:298-328 examples that the code satisfies
    assert orc.tau_schedule(32.0, 8192) == 256
    assert orc.stage_count(32, 16, 1.0) == 2
    for L, l, q, st in g["stage_count"]:
        assert orc.stage_count(L, l, q) == st
    ok, qm = orc.check_parameter_bounds(0.3, 4)
    assert ok is True and float.hex(qm) == g["check_parameter_bounds"][0][3]
    assert abs(qm - 0.3819718634) < 1e-9
    for s, n, inv in g["mod_inverse"]:
        assert orc.mod_inverse(s, n) == inv
    for u, L, b, want in g["bucket_of"]:
        assert orc.bucket_of(u, L, b) == want
    for key in ("random_params", "random_params_big"):
        rp = g[key]
        s, si = orc.random_params(rp["n"], rp["seed"], len(rp["sigma"]))
        assert list(s) == rp["sigma"] and list(si) == rp["sigma_inv"]
    for v, want in g["splitmix64"]:
        assert orc.splitmix64(v) == want
    for n, k, dl, b in g["initial_bucket_count"]:
        assert orc.initial_bucket_count(n, k, dl) == b


def test_windows_bit_exact(orc, golden):
    g = golden("windows")
    for rec in g["ok"]:
        w, taps = orc.window(rec["n"], rec["b"], rec["delta"])
        assert w == rec["w"]
        assert hashlib.sha256(taps.astype("<f8").tobytes()).hexdigest() == rec["taps_sha256"]
        offs = [a for a, _ in rec["response"]]
        got = orc.response_at(rec["n"], rec["b"], rec["delta"], offs)
        for (a, hv), v in zip(rec["response"], got):
            assert float.hex(float(v)) == hv, (rec["n"], rec["b"], a)


def test_window_errors(orc, golden):
    from oracle import OracleError
    for rec in golden("windows")["error"]:
        with pytest.raises(OracleError) as ei:
            orc.window(rec["n"], rec["b"], rec["delta"])
        assert ei.value.kind == "invalid_argument"
        assert str(ei.value) == rec["msg"]


def test_sfft4_small_bit_exact(orc, golden):
    from oracle import OracleError
    for rec in golden("sfft4_small"):
        x = make_signal(orc, rec).astype(np.complex128)
        if "error" in rec:
            with pytest.raises(OracleError) as ei:
                orc.sfft4(x, rec["k"], rec["l"], rec["q"], rec["algo_seed"], rec["delta"])
            assert str(ei.value) == rec["error"]["msg"]
            continue
        r = orc.sfft4(x, rec["k"], rec["l"], rec["q"], rec["algo_seed"], rec["delta"])
        f, c, stats = golden_result(rec)
        assert np.array_equal(r.f, f), (rec["n"], rec["k"], rec["seed"])
        assert np.array_equal(r.c.view(np.float64), c.view(np.float64))
        for key, v in stats.items():
            assert r.stats[key] == v, key


def test_trace_replays_sfft4(orc):
    """The per-stage trace (a replay of run_iteration) equals sfft4 bitwise."""
    x, _, _ = orc.generate_test_signal(1 << 14, 20, 77)
    r = orc.sfft4(x, 20, 16, 1.0, 5, 1e-8)
    tr = orc.sfft4_trace(x, 20, 16, 1.0, 5, 1e-8)
    assert np.array_equal(tr["result"].f, r.f)
    assert np.array_equal(tr["result"].c, r.c)
    # iteration 0 has nothing to subtract
    b0, r0 = tr["plan"].b[0], tr["plan"].rounds[0]
    assert np.array_equal(tr["pre"][: b0 * r0], tr["post"][: b0 * r0])
