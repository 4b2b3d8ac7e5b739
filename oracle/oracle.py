"""ctypes front end for the two CPU oracles (TEST INFRASTRUCTURE ONLY).

``load("reference")`` opens ``oracle/_ref/libmsfft_ref.so`` -- the reference
library compiled from /root/reference by ``oracle/Makefile``;
``load("port")`` opens ``oracle/_port/libmsfft_port.so`` -- the independent
restatement in ``oracle/port/``.  Both implement ``oracle_api.h``.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "reference": os.path.join(HERE, "_ref", "libmsfft_ref.so"),
    "port": os.path.join(HERE, "_port", "libmsfft_port.so"),
}
MAX_ITERS = 64
MAX_ROUNDS = 512

i64, u64, f64, i32 = C.c_int64, C.c_uint64, C.c_double, C.c_int32
P = C.POINTER


class OracleError(Exception):
    """Raised for a non-zero oracle status; ``kind`` is invalid_argument,
    domain_error or other (the reference exception class)."""

    def __init__(self, kind: str, msg: str):
        super().__init__(msg)
        self.kind = kind


class _Plan(C.Structure):
    _fields_ = [
        ("iterations", i32),
        ("b_first", i64),
        ("b", i64 * MAX_ITERS),
        ("w", i64 * MAX_ITERS),
        ("rounds", i32 * MAX_ITERS),
        ("k_m", i64 * MAX_ITERS),
        ("budget", i64 * MAX_ITERS),
        ("sigma", i64 * MAX_ITERS),
        ("sigma_inv", i64 * MAX_ITERS),
        ("taus", i64 * MAX_ROUNDS),
    ]


@dataclass
class Plan:
    iterations: int
    b_first: int
    b: list
    w: list
    rounds: list
    k_m: list
    budget: list
    sigma: list
    sigma_inv: list
    taus: list  # list of lists, one per iteration


@dataclass
class Result:
    f: np.ndarray  # int64 ascending
    c: np.ndarray  # complex128
    stats: dict = field(default_factory=dict)

    def as_dict(self):
        return {int(a): complex(b) for a, b in zip(self.f, self.c)}


def available(kind: str) -> bool:
    return os.path.exists(LIBS[kind])


_cache: dict = {}


def load(kind: str = "reference") -> "Oracle":
    if kind not in _cache:
        _cache[kind] = Oracle(kind)
    return _cache[kind]


def _ptr(a, ct):
    return a.ctypes.data_as(P(ct))


def _cx(x) -> np.ndarray:
    """complex array -> contiguous interleaved float64 view."""
    x = np.ascontiguousarray(np.asarray(x, dtype=np.complex128))
    return x.view(np.float64)


class Oracle:
    def __init__(self, kind: str):
        path = LIBS[kind]
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library missing: {path} (run `make -C oracle`)")
        self.kind = kind
        L = self.lib = C.CDLL(path)
        E = [C.c_char_p, i64]
        L.orc_kind.restype = C.c_char_p
        L.orc_splitmix64.argtypes, L.orc_splitmix64.restype = [u64], u64
        L.orc_mod_inverse.argtypes = [i64, i64, P(i64)] + E
        L.orc_bucket_of.argtypes, L.orc_bucket_of.restype = [i64, i64, i64], i64
        L.orc_tau_schedule.argtypes, L.orc_tau_schedule.restype = [f64, i64], i64
        L.orc_stage_count.argtypes, L.orc_stage_count.restype = [f64, i64, f64], C.c_int
        L.orc_check_parameter_bounds.argtypes = [f64, i64, f64, P(C.c_int), P(f64)] + E
        L.orc_cfg_validate.argtypes = [i64, f64] + E
        L.orc_random_params.argtypes = [i64, u64, i64, P(i64), P(i64)] + E
        L.orc_initial_bucket_count.argtypes = [i64, i64, f64, P(i64)] + E
        L.orc_plan_build.argtypes = [i64, i64, i64, f64, u64, f64, P(_Plan)] + E
        L.orc_window.argtypes = [i64, i64, f64, P(i64), P(f64), i64] + E
        L.orc_response_at.argtypes = [i64, i64, f64, P(i64), i64, P(f64)] + E
        L.orc_bucketize.argtypes = [i64, P(f64), i64, f64, i64, i64, P(f64)] + E
        L.orc_predict.argtypes = [i64, i64, f64, i64, P(i64), P(f64), i64, i64, P(f64)] + E
        L.orc_locate.argtypes = [i64, i64, f64, i64, f64, i64, i64, P(i64), P(f64), P(i64),
                                 P(C.c_int)] + E
        L.orc_estimate_value.argtypes = [i64, i64, f64, f64, f64, i64, P(f64)] + E
        L.orc_sfft4.argtypes = [i64, P(f64), i64, i64, f64, u64, f64, i64, P(i64), P(f64),
                                P(i64), P(i64), P(f64)] + E
        L.orc_sfft4_trace.argtypes = [i64, P(f64), i64, i64, f64, u64, f64, P(f64), P(f64),
                                      P(i64), P(i64), P(i32), P(f64), P(i64), i64, P(i64),
                                      P(f64), P(i64)] + E
        L.orc_sfft4_batch_c64.argtypes = [i64, i64, P(C.c_float), i64, i64, f64, P(u64), f64,
                                          C.c_int, i64, P(i64), P(f64), P(i64), P(f64)] + E
        L.orc_generate_test_signal.argtypes = [i64, i64, u64, P(f64), P(i64), P(f64)] + E
        L.orc_add_awgn.argtypes = [i64, P(f64), f64, u64] + E
        L.orc_dft_dense.argtypes = [i64, P(f64), P(f64)] + E
        L.orc_idft_dense.argtypes = [i64, P(f64), P(f64)] + E
        L.orc_synthesize.argtypes = [i64, i64, P(i64), P(f64), P(f64)] + E
        L.orc_error_metrics.argtypes = [i64, i64, P(i64), P(f64), i64, P(i64), P(f64), i64,
                                        P(i64), P(f64), P(f64)] + E
        L.orc_top_k_spectrum.argtypes = [i64, P(f64), i64, P(i64), P(f64), P(i64)] + E
        L.orc_write_signal_file.argtypes = [C.c_char_p, i64, P(f64)] + E
        L.orc_read_signal_file.argtypes = [C.c_char_p, i64, P(f64), P(i64)] + E
        L.orc_write_truth_csv.argtypes = [C.c_char_p, i64, i64, P(i64), P(f64)] + E
        L.orc_read_truth_csv.argtypes = [C.c_char_p, i64, i64, P(i64), P(f64), P(i64)] + E
        if hasattr(L, "orc_phase_experiment"):
            L.orc_phase_experiment.argtypes = [i64, i64, i64, P(f64), i64, i64, u64, P(f64)] + E
            L.orc_phase_trials.argtypes = [i64, i64, i64, f64, i64, i64, u64, P(i64), P(f64)] + E
            L.orc_phase_experiment.restype = C.c_int
            L.orc_phase_trials.restype = C.c_int
        for fn in ("orc_mod_inverse", "orc_check_parameter_bounds", "orc_cfg_validate",
                   "orc_random_params", "orc_initial_bucket_count", "orc_plan_build",
                   "orc_window", "orc_response_at", "orc_bucketize", "orc_predict", "orc_locate",
                   "orc_estimate_value", "orc_sfft4", "orc_sfft4_trace", "orc_sfft4_batch_c64",
                   "orc_generate_test_signal", "orc_add_awgn", "orc_dft_dense",
                   "orc_idft_dense", "orc_synthesize", "orc_error_metrics", "orc_top_k_spectrum",
                   "orc_write_signal_file", "orc_read_signal_file", "orc_write_truth_csv",
                   "orc_read_truth_csv"):
            getattr(L, fn).restype = C.c_int

    # -- error plumbing ------------------------------------------------------
    def _call(self, fn, *args):
        err = C.create_string_buffer(512)
        st = fn(*args, err, 512)
        if st != 0:
            kind = {1: "invalid_argument", 2: "domain_error"}.get(st, "other")
            raise OracleError(kind, err.value.decode())
        return st

    # -- scalars -------------------------------------------------------------
    def splitmix64(self, x: int) -> int:
        return int(self.lib.orc_splitmix64(x & (2**64 - 1)))

    def mod_inverse(self, sigma: int, n: int) -> int:
        out = i64()
        self._call(self.lib.orc_mod_inverse, sigma, n, C.byref(out))
        return out.value

    def bucket_of(self, u, L, b):
        return int(self.lib.orc_bucket_of(u, L, b))

    def tau_schedule(self, length, n):
        return int(self.lib.orc_tau_schedule(float(length), n))

    def stage_count(self, length, l, q):
        return int(self.lib.orc_stage_count(float(length), l, float(q)))

    def check_parameter_bounds(self, max_dphi, l, q=0.0):
        ok, qm = C.c_int(), f64()
        self._call(self.lib.orc_check_parameter_bounds, float(max_dphi), l, float(q),
                   C.byref(ok), C.byref(qm))
        return bool(ok.value), qm.value

    def cfg_validate(self, l, q):
        self._call(self.lib.orc_cfg_validate, l, float(q))

    def random_params(self, n, seed, count):
        s = np.zeros(count, np.int64)
        si = np.zeros(count, np.int64)
        self._call(self.lib.orc_random_params, n, seed, count, _ptr(s, i64), _ptr(si, i64))
        return s, si

    def initial_bucket_count(self, n, k, delta):
        out = i64()
        self._call(self.lib.orc_initial_bucket_count, n, k, float(delta), C.byref(out))
        return out.value

    def plan(self, n, k, l=16, q=1.0, seed=0, delta=1e-8) -> Plan:
        p = _Plan()
        self._call(self.lib.orc_plan_build, n, k, l, float(q), seed, float(delta), C.byref(p))
        it = p.iterations
        taus, off = [], 0
        for m in range(it):
            taus.append([p.taus[off + r] for r in range(p.rounds[m])])
            off += p.rounds[m]
        return Plan(it, p.b_first, list(p.b[:it]), list(p.w[:it]), list(p.rounds[:it]),
                    list(p.k_m[:it]), list(p.budget[:it]), list(p.sigma[:it]),
                    list(p.sigma_inv[:it]), taus)

    # -- window ----------------------------------------------------------------
    def window(self, n, b, delta, taps=True):
        w = i64()
        self._call(self.lib.orc_window, n, b, float(delta), C.byref(w), None, 0)
        if not taps:
            return w.value, None
        g = np.zeros(w.value, np.float64)
        self._call(self.lib.orc_window, n, b, float(delta), C.byref(w), _ptr(g, f64), w.value)
        return w.value, g

    def response_at(self, n, b, delta, idx):
        idx = np.ascontiguousarray(np.asarray(idx, dtype=np.int64))
        out = np.zeros(idx.size, np.float64)
        self._call(self.lib.orc_response_at, n, b, float(delta), _ptr(idx, i64), idx.size,
                   _ptr(out, f64))
        return out

    # -- bucketization -----------------------------------------------------------
    def bucketize(self, x, b, delta, sigma, tau):
        xv = _cx(x)
        n = xv.size // 2
        out = np.zeros(2 * b, np.float64)
        self._call(self.lib.orc_bucketize, n, _ptr(xv, f64), b, float(delta), sigma, tau,
                   _ptr(out, f64))
        return out.view(np.complex128)

    def predict(self, n, b, delta, f, c, sigma, tau):
        f = np.ascontiguousarray(np.asarray(f, dtype=np.int64))
        cv = _cx(c)
        out = np.zeros(2 * b, np.float64)
        self._call(self.lib.orc_predict, n, b, float(delta), f.size, _ptr(f, i64), _ptr(cv, f64),
                   sigma, tau, _ptr(out, f64))
        return out.view(np.complex128)

    def locate(self, n, b, delta, l, q, bucket, taus, rounds):
        taus = np.ascontiguousarray(np.asarray(taus, dtype=np.int64))
        rv = _cx(np.asarray(rounds).reshape(-1))
        u, st = i64(), C.c_int()
        self._call(self.lib.orc_locate, n, b, float(delta), l, float(q), bucket, taus.size,
                   _ptr(taus, i64), _ptr(rv, f64), C.byref(u), C.byref(st))
        return (None if u.value < 0 else u.value), st.value

    def estimate_value(self, n, b, delta, y, u):
        out = np.zeros(2, np.float64)
        self._call(self.lib.orc_estimate_value, n, b, float(delta), float(y.real), float(y.imag),
                   u, _ptr(out, f64))
        return complex(out[0], out[1])

    # -- full transform ------------------------------------------------------------
    def sfft4(self, x, k, l=16, q=1.0, seed=0, delta=1e-8) -> Result:
        xv = _cx(x)
        n = xv.size // 2
        cap = max(k, 1)
        f = np.zeros(cap, np.int64)
        c = np.zeros(2 * cap, np.float64)
        cnt = i64()
        si = np.zeros(4 + MAX_ITERS, np.int64)
        sd = np.zeros(2, np.float64)
        self._call(self.lib.orc_sfft4, n, _ptr(xv, f64), k, l, float(q), seed, float(delta), cap,
                   _ptr(f, i64), _ptr(c, f64), C.byref(cnt), _ptr(si, i64), _ptr(sd, f64))
        m = cnt.value
        it = int(si[2])
        stats = dict(samples_used=int(si[0]), samples_round_sum=int(si[1]), iterations=it,
                     b_first=int(si[3]), stage_counts=[int(v) for v in si[4:4 + it]],
                     sample_fraction=float(sd[0]), runtime_ms=float(sd[1]))
        return Result(f[:m].copy(), c.view(np.complex128)[:m].copy(), stats)

    def sfft4_trace(self, x, k, l=16, q=1.0, seed=0, delta=1e-8):
        xv = _cx(x)
        n = xv.size // 2
        plan = self.plan(n, k, l, q, seed, delta)
        nv = sum(r * b for r, b in zip(plan.rounds, plan.b))
        ns = sum(plan.budget)
        pre = np.zeros(2 * nv, np.float64)
        post = np.zeros(2 * nv, np.float64)
        sb = np.zeros(ns, np.int64)
        su = np.zeros(ns, np.int64)
        ss = np.zeros(ns, np.int32)
        sv = np.zeros(2 * ns, np.float64)
        sf = np.zeros(ns, np.int64)
        cap = max(k, 1)
        f = np.zeros(cap, np.int64)
        c = np.zeros(2 * cap, np.float64)
        cnt = i64()
        self._call(self.lib.orc_sfft4_trace, n, _ptr(xv, f64), k, l, float(q), seed,
                   float(delta), _ptr(pre, f64), _ptr(post, f64), _ptr(sb, i64), _ptr(su, i64),
                   _ptr(ss, i32), _ptr(sv, f64), _ptr(sf, i64), cap, _ptr(f, i64),
                   _ptr(c, f64), C.byref(cnt))
        m = cnt.value
        return dict(plan=plan, pre=pre.view(np.complex128), post=post.view(np.complex128),
                    sel_bucket=sb, sel_u=su, sel_status=ss, sel_value=sv.view(np.complex128),
                    sel_f=sf, result=Result(f[:m].copy(), c.view(np.complex128)[:m].copy()))

    def sfft4_batch_c64(self, x, k, l, q, seeds, delta, threads):
        """x: (nsig, n) complex64.  Returns (list of Result, wall_ms)."""
        x = np.ascontiguousarray(np.asarray(x, dtype=np.complex64))
        nsig, n = x.shape
        xv = x.view(np.float32)
        seeds = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64))
        cap = max(k, 1)
        f = np.zeros((nsig, cap), np.int64)
        c = np.zeros((nsig, 2 * cap), np.float64)
        cnt = np.zeros(nsig, np.int64)
        wall = f64()
        self._call(self.lib.orc_sfft4_batch_c64, nsig, n, _ptr(xv, C.c_float), k, l, float(q),
                   _ptr(seeds, u64), float(delta), int(threads), cap, _ptr(f, i64), _ptr(c, f64),
                   _ptr(cnt, i64), C.byref(wall))
        cc = c.view(np.complex128)
        out = [Result(f[i, :cnt[i]].copy(), cc[i, :cnt[i]].copy()) for i in range(nsig)]
        return out, wall.value

    # -- signal model ----------------------------------------------------------------
    def generate_test_signal(self, n, k, seed):
        x = np.zeros(2 * n, np.float64)
        f = np.zeros(k, np.int64)
        c = np.zeros(2 * k, np.float64)
        self._call(self.lib.orc_generate_test_signal, n, k, seed, _ptr(x, f64), _ptr(f, i64),
                   _ptr(c, f64))
        return x.view(np.complex128), f, c.view(np.complex128)

    def add_awgn(self, x, snr_db, seed):
        xv = _cx(x).copy()
        n = xv.size // 2
        self._call(self.lib.orc_add_awgn, n, _ptr(xv, f64), float(snr_db), seed)
        return xv.view(np.complex128)

    # -- signal helpers --------------------------------
    def dft_dense(self, x):
        xv = _cx(x)
        out = np.zeros_like(xv)
        self._call(self.lib.orc_dft_dense, xv.size // 2, _ptr(xv, f64), _ptr(out, f64))
        return out.view(np.complex128)

    def idft_dense(self, spec):
        sv = _cx(spec)
        out = np.zeros_like(sv)
        self._call(self.lib.orc_idft_dense, sv.size // 2, _ptr(sv, f64), _ptr(out, f64))
        return out.view(np.complex128)

    def synthesize(self, n, f, c):
        f = np.ascontiguousarray(np.asarray(f, dtype=np.int64))
        cv = _cx(c)
        x = np.zeros(2 * n, np.float64)
        self._call(self.lib.orc_synthesize, n, f.size, _ptr(f, i64), _ptr(cv, f64), _ptr(x, f64))
        return x.view(np.complex128)

    def error_metrics(self, n, tf, tc, ef, ec, k):
        tf = np.ascontiguousarray(np.asarray(tf, dtype=np.int64))
        ef = np.ascontiguousarray(np.asarray(ef, dtype=np.int64))
        tcv, ecv = _cx(tc), _cx(ec)
        l0, l1, l2 = i64(), f64(), f64()
        self._call(self.lib.orc_error_metrics, n, tf.size, _ptr(tf, i64), _ptr(tcv, f64),
                   ef.size, _ptr(ef, i64), _ptr(ecv, f64), k, C.byref(l0), C.byref(l1),
                   C.byref(l2))
        return l0.value, l1.value, l2.value

    def top_k_spectrum(self, spec, k):
        sv = _cx(spec)
        n = sv.size // 2
        f = np.zeros(max(k, 1), np.int64)
        c = np.zeros(2 * max(k, 1), np.float64)
        cnt = i64()
        self._call(self.lib.orc_top_k_spectrum, n, _ptr(sv, f64), k, _ptr(f, i64), _ptr(c, f64),
                   C.byref(cnt))
        return f[:cnt.value], c.view(np.complex128)[:cnt.value]

    def write_signal_file(self, path, x):
        xv = _cx(x)
        self._call(self.lib.orc_write_signal_file, str(path).encode(), xv.size // 2,
                   _ptr(xv, f64))

    def read_signal_file(self, path, cap=1 << 24):
        x = np.zeros(2 * cap, np.float64)
        n = i64()
        self._call(self.lib.orc_read_signal_file, str(path).encode(), cap, _ptr(x, f64),
                   C.byref(n))
        if n.value > cap:
            return self.read_signal_file(path, n.value)
        return x.view(np.complex128)[:n.value].copy()

    def write_truth_csv(self, path, n, f, c):
        f = np.ascontiguousarray(np.asarray(f, dtype=np.int64))
        cv = _cx(c)
        self._call(self.lib.orc_write_truth_csv, str(path).encode(), n, f.size, _ptr(f, i64),
                   _ptr(cv, f64))

    def read_truth_csv(self, path, n, cap=1 << 20):
        f = np.zeros(cap, np.int64)
        c = np.zeros(2 * cap, np.float64)
        cnt = i64()
        self._call(self.lib.orc_read_truth_csv, str(path).encode(), n, cap, _ptr(f, i64),
                   _ptr(c, f64), C.byref(cnt))
        return f[:cnt.value].copy(), c.view(np.complex128)[:cnt.value].copy()

    # -- phase-error Monte Carlo (reference only) --------------------------------
    def phase_experiment(self, n, k, b, snr_list, trials, seed):
        """-> list of dicts {bin_mass (70), p50, p99, max} per SNR."""
        if not hasattr(self.lib, "orc_phase_experiment"):
            raise OracleError("other", "phase_mc is not in this oracle")
        snr = np.ascontiguousarray(np.asarray(snr_list, dtype=np.float64))
        out = np.zeros(73 * snr.size, np.float64)
        self._call(self.lib.orc_phase_experiment, n, k, b, _ptr(snr, f64), snr.size, trials,
                   seed, _ptr(out, f64))
        out = out.reshape(-1, 73)
        return [{"bin_mass": r[:70].copy(), "p50": r[70], "p99": r[71], "max": r[72]} for r in out]

    def phase_trials(self, n, k, b, snr, si, trials, seed):
        """Accepted trials of SNR index si: (ints [t,3] u/bucket/tau, doubles [t,7])."""
        oi = np.zeros(3 * trials, np.int64)
        od = np.zeros(7 * trials, np.float64)
        self._call(self.lib.orc_phase_trials, n, k, b, float(snr), si, trials, seed,
                   _ptr(oi, i64), _ptr(od, f64))
        return oi.reshape(-1, 3), od.reshape(-1, 7)
