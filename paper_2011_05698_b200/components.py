"""The reference's component API on the sfft4 path: the
functions its own tests call directly, each on the GPU through the C ABI.

    bucketize         proj/src/bucketize.cpp:50-61 (bucketize.hpp:63-86)
    predict_buckets   proj/src/bucketize.cpp:70-95
    subtract          proj/src/bucketize.cpp:97-104 (host, elementwise)
    locate_frequency  proj/src/locate.cpp:83-123
    estimate_value    proj/src/sfft4.cpp:27-36
    run_iteration     proj/src/sfft4.cpp:38-113 (composed from the above)

Types mirror the reference: PermutationParams (bucketize.hpp:16-20),
BucketSet (:24-30), LocateOutcome (locate.hpp:42-45), and FlatWindow as a
handle on the device window cache (n, b, delta; window.hpp:16-30).  The
batched forms (bucketize_rounds, locate_frequencies, estimate_values) are the
same functions over many rounds / buckets in one launch.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import DomainError, InvalidArgument, MultiscaleConfig, SparseSpectrum, _raise
from . import _lib as _L
from .signal import _buf

__all__ = ["FlatWindow", "PermutationParams", "BucketSet", "LocateOutcome", "flat_window",
           "bucketize", "bucketize_rounds", "predict_buckets", "subtract", "locate_frequency",
           "locate_frequencies", "estimate_value", "estimate_values", "tau_plan", "sigma_plan",
           "Rng", "IterationState", "run_iteration"]


def _err():
    return C.create_string_buffer(1024)


@dataclass(frozen=True)
class FlatWindow:
    """Handle on the designed window (n, b, delta); w = support."""
    n: int
    b: int
    delta: float
    w: int

    @property
    def l_width(self) -> int:
        return self.n // self.b


def flat_window(n: int, b: int, delta: float) -> FlatWindow:
    """get_flat_window (window.cpp:179-193): designs (or reuses) the window on
    the current device; infeasible parameters raise the reference's errors."""
    from . import window
    w, _ = window(n, b, delta)
    return FlatWindow(int(n), int(b), float(delta), int(w))


@dataclass(frozen=True)
class PermutationParams:
    sigma: int
    sigma_inv: int = 0
    tau: int = 0


@dataclass
class BucketSet:
    n: int
    b: int
    values: np.ndarray                 # complex128 [b]
    params: PermutationParams = field(default_factory=PermutationParams)
    samples_read: int = 0


@dataclass(frozen=True)
class LocateOutcome:
    u: int
    stages: int


def _cx_host(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.complex128))


def bucketize_rounds(x, win: FlatWindow, params) -> list[BucketSet]:
    """bucketize of one signal x (numpy or CUDA torch, complex64/128, n
    samples) under every PermutationParams in `params`, in one launch."""
    params = list(params)
    ptr, loc, code, keep = _buf(x)
    if code is None:
        raise InvalidArgument("bucketize: x must be complex")
    n = int(keep.shape[-1])
    if n != win.n:
        raise InvalidArgument("bucketize: signal/window size mismatch")
    sig = np.array([p.sigma for p in params], np.int64)
    tau = np.array([p.tau for p in params], np.int64)
    out = np.zeros((len(params), win.b), np.complex128)
    w = C.c_int64()
    e = _err()
    _raise(_L.lib().msfft_bucketize(ptr, n, code, loc, win.b, win.delta,
                                    C.c_void_p(sig.ctypes.data), C.c_void_p(tau.ctypes.data),
                                    len(params), C.c_void_p(out.ctypes.data), _L.MSFFT_HOST,
                                    C.byref(w), e, 1024), e)
    return [BucketSet(n, win.b, out[r], p, int(w.value)) for r, p in enumerate(params)]


def bucketize(x, win: FlatWindow, params: PermutationParams) -> BucketSet:
    return bucketize_rounds(x, win, [params])[0]


def predict_buckets(known: SparseSpectrum, win: FlatWindow, params) -> BucketSet | list:
    """predict_buckets for one PermutationParams (-> BucketSet) or a list of
    them (-> list, one launch)."""
    if known.n != win.n:
        raise InvalidArgument("predict_buckets: size mismatch")
    many = isinstance(params, (list, tuple))
    plist = list(params) if many else [params]
    f = np.ascontiguousarray(np.asarray(known.positions, np.int64))
    c = _cx_host(known.coeffs)
    sig = np.array([p.sigma for p in plist], np.int64)
    tau = np.array([p.tau for p in plist], np.int64)
    out = np.zeros((len(plist), win.b), np.complex128)
    e = _err()
    _raise(_L.lib().msfft_predict_buckets(win.n, win.b, win.delta, C.c_void_p(f.ctypes.data),
                                          C.c_void_p(c.ctypes.data), f.size,
                                          C.c_void_p(sig.ctypes.data),
                                          C.c_void_p(tau.ctypes.data), len(plist),
                                          C.c_void_p(out.ctypes.data), _L.MSFFT_HOST, e, 1024), e)
    sets = [BucketSet(win.n, win.b, out[r], p, 0) for r, p in enumerate(plist)]
    return sets if many else sets[0]


def subtract(a: BucketSet, b_set: BucketSet) -> BucketSet:
    """bucketize.cpp:97-104."""
    if (a.b != b_set.b or a.n != b_set.n or a.params.sigma != b_set.params.sigma or
            a.params.tau != b_set.params.tau):
        raise InvalidArgument("subtract: bucket sets are not from the same round")
    return BucketSet(a.n, a.b, np.asarray(a.values) - np.asarray(b_set.values), a.params,
                     a.samples_read)


def locate_frequencies(buckets, rounds: list[BucketSet], cfg: MultiscaleConfig,
                       win: FlatWindow) -> list:
    """locate_frequency for every bucket in `buckets` against one round set
    (one launch): a LocateOutcome or None (nullopt) per bucket."""
    cfg = cfg or MultiscaleConfig()
    bk = np.ascontiguousarray(np.asarray(list(buckets), np.int64))
    if not rounds:
        raise InvalidArgument("locate_frequency: no rounds")
    vals = np.ascontiguousarray(np.stack([_cx_host(r.values) for r in rounds]))
    tau = np.array([r.params.tau for r in rounds], np.int64)
    u = np.zeros(bk.size, np.int64)
    st = np.zeros(bk.size, np.int32)
    status = np.zeros(bk.size, np.int32)
    e = _err()
    _raise(_L.lib().msfft_locate_frequency(win.n, win.b, int(cfg.l), float(cfg.q),
                                           C.c_void_p(bk.ctypes.data), bk.size,
                                           C.c_void_p(vals.ctypes.data),
                                           C.c_void_p(tau.ctypes.data), len(rounds),
                                           C.c_void_p(u.ctypes.data), C.c_void_p(st.ctypes.data),
                                           C.c_void_p(status.ctypes.data), _L.MSFFT_HOST, e,
                                           1024), e)
    return [LocateOutcome(int(u[i]), int(st[i])) if status[i] == 0 else None
            for i in range(bk.size)]


def locate_frequency(bucket: int, rounds: list[BucketSet], cfg: MultiscaleConfig,
                     win: FlatWindow):
    return locate_frequencies([bucket], rounds, cfg, win)[0]


def estimate_values(y0, u, win: FlatWindow):
    """estimate_value over arrays: (values, ok) with ok False where the
    reference throws (|G| < 0.5)."""
    y = _cx_host(np.atleast_1d(y0))
    uu = np.ascontiguousarray(np.atleast_1d(np.asarray(u, np.int64)))
    out = np.zeros(y.size, np.complex128)
    status = np.zeros(y.size, np.int32)
    e = _err()
    _raise(_L.lib().msfft_estimate_values(win.n, win.b, win.delta, C.c_void_p(y.ctypes.data),
                                          C.c_void_p(uu.ctypes.data), y.size,
                                          C.c_void_p(out.ctypes.data),
                                          C.c_void_p(status.ctypes.data), _L.MSFFT_HOST, e,
                                          1024), e)
    return out, status == 0


def estimate_value(y0: complex, u: int, win: FlatWindow) -> complex:
    v, ok = estimate_values([y0], [u], win)
    if not ok[0]:
        raise DomainError("estimate_value: located position outside the pass region")
    return complex(v[0])


def tau_plan(l_width: int, n: int, cfg: MultiscaleConfig | None = None) -> list[int]:
    """{0, tau_1..tau_R} of an iteration (stage_count + tau_schedule,
    sfft4.cpp:49-55), host-side like the reference."""
    cfg = cfg or MultiscaleConfig()
    taus = np.zeros(64, np.int64)
    rounds = C.c_int32()
    e = _err()
    _raise(_L.lib().msfft_tau_plan(float(l_width), int(n), int(cfg.l), float(cfg.q),
                                   taus.ctypes.data_as(C.POINTER(C.c_int64)), taus.size,
                                   C.byref(rounds), e, 1024), e)
    return [int(t) for t in taus[:rounds.value]]


def sigma_plan(seed: int, n: int, iterations: int) -> list[PermutationParams]:
    """random_params(n, Rng(seed), 0) for the first `iterations` iterations
    of a transform seeded `seed` (bucketize.cpp:39-48, sfft4.cpp:48)."""
    s = np.zeros(iterations, np.int64)
    si = np.zeros(iterations, np.int64)
    e = _err()
    _raise(_L.lib().msfft_sigma_plan(int(seed) & (2**64 - 1), int(n), int(iterations),
                                     s.ctypes.data_as(C.POINTER(C.c_int64)),
                                     si.ctypes.data_as(C.POINTER(C.c_int64)), e, 1024), e)
    return [PermutationParams(int(a), int(b), 0) for a, b in zip(s, si)]


# ---- scalar helpers (host plan code) and locate arithmetic (device) ---------

def mod_inverse(sigma: int, n: int) -> int:
    """bucketize.cpp:21-37."""
    out = C.c_int64()
    e = _err()
    _raise(_L.lib().msfft_mod_inverse(int(sigma), int(n), C.byref(out), e, 1024), e)
    return out.value


def bucket_of(u: int, l_width: int, b: int) -> int:
    """bucketize.cpp:63-68: round(u/L) mod b, ties away from zero."""
    return int(_L.lib().msfft_bucket_of(int(u), int(l_width), int(b)))


def stage_count(region_length: float, cfg: MultiscaleConfig | None = None) -> int:
    """locate.cpp:44-53."""
    cfg = cfg or MultiscaleConfig()
    out = C.c_int32()
    e = _err()
    _raise(_L.lib().msfft_stage_count(float(region_length), int(cfg.l), float(cfg.q),
                                      C.byref(out), e, 1024), e)
    return out.value


def tau_schedule(region_length: float, n: int) -> int:
    """locate.cpp:39-42."""
    out = C.c_int64()
    e = _err()
    _raise(_L.lib().msfft_tau_schedule(float(region_length), int(n), C.byref(out), e, 1024), e)
    return out.value


def initial_bucket_count(n: int, k: int, delta: float) -> int:
    """sfft4.cpp:115-129 (windows designed on the GPU)."""
    out = C.c_int64()
    e = _err()
    _raise(_L.lib().msfft_initial_bucket_count(int(n), int(k), float(delta), C.byref(out), e,
                                               1024), e)
    return out.value


def check_parameter_bounds(max_dphi: float, l: int, q: float = 0.0):
    """locate.cpp:125-132 -> (l_ok, q_min)."""
    ok, qm = C.c_int32(), C.c_double()
    e = _err()
    _raise(_L.lib().msfft_check_parameter_bounds(float(max_dphi), int(l), float(q), C.byref(ok),
                                                 C.byref(qm), e, 1024), e)
    return bool(ok.value), qm.value


def phase_of(z):
    """phase_of (locate.cpp:32-37) of each complex z on the device (the
    decode's arithmetic): (phases, status) with status 1 where z == 0."""
    z = np.ascontiguousarray(np.atleast_1d(np.asarray(z, np.complex128)))
    ph = np.zeros(z.size, np.float64)
    st = np.zeros(z.size, np.int32)
    e = _err()
    _raise(_L.lib().msfft_phase_of(C.c_void_p(z.ctypes.data), z.size, C.c_void_p(ph.ctypes.data),
                                   C.c_void_p(st.ctypes.data), e, 1024), e)
    return ph, st


def position_phase(u, tau, n: int) -> np.ndarray:
    """position_phase (locate.cpp:19-23), elementwise on the device."""
    u = np.ascontiguousarray(np.atleast_1d(np.asarray(u, np.float64)))
    tau = np.ascontiguousarray(np.broadcast_to(np.asarray(tau, np.int64), u.shape))
    out = np.zeros(u.size, np.float64)
    e = _err()
    _raise(_L.lib().msfft_position_phase(C.c_void_p(u.ctypes.data), C.c_void_p(tau.ctypes.data),
                                         u.size, int(n), C.c_void_p(out.ctypes.data), e, 1024), e)
    return out


def circular_phase_distance(a, b) -> np.ndarray:
    """circular_phase_distance (locate.cpp:14-17), elementwise on the device."""
    a = np.ascontiguousarray(np.atleast_1d(np.asarray(a, np.float64)))
    b = np.ascontiguousarray(np.broadcast_to(np.asarray(b, np.float64), a.shape))
    out = np.zeros(a.size, np.float64)
    e = _err()
    _raise(_L.lib().msfft_circular_phase_distance(C.c_void_p(a.ctypes.data),
                                                  C.c_void_p(b.ctypes.data), a.size,
                                                  C.c_void_p(out.ctypes.data), e, 1024), e)
    return out


_REGION = np.dtype([("u_min", np.float64), ("length", np.float64), ("stage", np.int32),
                    ("reserved", np.int32)])


def locate_step(phi, tau, u_min, length, stage, cfg: MultiscaleConfig, n: int):
    """locate_step (locate.cpp:63-81) for arrays of (measurement, region):
    returns (u_min, length, stage) arrays of the next regions."""
    phi = np.ascontiguousarray(np.atleast_1d(np.asarray(phi, np.float64)))
    m = phi.size
    tau = np.ascontiguousarray(np.broadcast_to(np.asarray(tau, np.int64), (m,)))
    reg = np.zeros(m, _REGION)
    reg["u_min"], reg["length"], reg["stage"] = u_min, length, stage
    out = np.zeros(m, _REGION)
    e = _err()
    _raise(_L.lib().msfft_locate_step(C.c_void_p(phi.ctypes.data), C.c_void_p(tau.ctypes.data),
                                      C.c_void_p(reg.ctypes.data), m, int(cfg.l), float(cfg.q),
                                      int(n), C.c_void_p(out.ctypes.data), e, 1024), e)
    return out["u_min"].copy(), out["length"].copy(), out["stage"].copy()


def bucketize_fn(n: int, sample, win: FlatWindow, params: PermutationParams) -> BucketSet:
    """bucketize_fn<Sampler> (bucketize.hpp:63-86): `sample(idx)` is called
    once per tap in increasing tap order on this thread; the fold, DIT and
    1/n run on the GPU (bit-identical to the reference's loop)."""
    h = (win.w - 1) // 2
    mask = n - 1
    v = np.zeros(win.w, np.complex128)
    for t in range(-h, h + 1):
        v[h + t] = sample((params.sigma * ((t - params.tau) & mask)) & mask)
    out = np.zeros(win.b, np.complex128)
    w = C.c_int64()
    e = _err()
    _raise(_L.lib().msfft_bucketize_taps(int(n), int(win.b), float(win.delta),
                                         C.c_void_p(v.ctypes.data), 1,
                                         C.c_void_p(out.ctypes.data), C.byref(w), e, 1024), e)
    return BucketSet(n, win.b, out, params, int(w.value))


class Rng:
    """The draws sfft4 makes from its Rng (rng.hpp:19-59): one
    random_params(n, rng, 0) per iteration (sfft4.cpp:48), reproduced from
    the seed by the host σ plan."""

    def __init__(self, seed: int):
        self.seed = int(seed)
        self.draws = 0

    def random_params(self, n: int) -> PermutationParams:
        p = sigma_plan(self.seed, n, self.draws + 1)[self.draws]
        self.draws += 1
        return p


@dataclass
class IterationState:
    """sfft4.hpp:14-30; `accumulated` maps f -> c (ascending on read)."""
    m: int = 1
    k_m: int = 0
    b_m: int = 0
    delta: float = 1e-8
    accumulated: dict = field(default_factory=dict)
    sigma_m: int = 1
    tau_plan: list = field(default_factory=list)
    w_m: int = 0
    stages_m: int = 0
    samples_round_sum: int = 0


def run_iteration(x, state: IterationState, cfg: MultiscaleConfig, rng: Rng) -> SparseSpectrum:
    """run_iteration (sfft4.cpp:38-113) composed from the component API:
    encode every round, subtract the prediction of the accumulated tones,
    rank |y0|, locate and estimate the buckets above the threshold, fold the
    found tones into state.accumulated, halve k_m / b_m.  Returns the tones
    found this iteration.  Each step is one GPU launch over all rounds or
    all candidate buckets."""
    n = int(x.shape[-1])
    win = flat_window(n, state.b_m, state.delta)
    base = rng.random_params(n)
    taus = tau_plan(win.l_width, n, cfg)
    state.sigma_m, state.tau_plan, state.w_m, state.stages_m = base.sigma, taus, win.w, len(taus) - 1
    params = [PermutationParams(base.sigma, base.sigma_inv, t) for t in taus]
    rounds = bucketize_rounds(x, win, params)
    if state.accumulated:
        fs = np.array(sorted(state.accumulated), np.int64)
        known = SparseSpectrum(n, fs, np.array([state.accumulated[f] for f in fs]))
        rounds = [subtract(r, p) for r, p in zip(rounds, predict_buckets(known, win, params))]
    state.samples_round_sum += len(taus) * win.w
    budget = min(state.k_m, state.b_m)
    y0 = rounds[0].values
    mag = np.abs(y0)  # hypot, as std::abs(cplx)
    order = np.argsort(-mag, kind="stable")
    threshold = 0.2 * mag[order[budget - 1]]
    cand = [int(order[r]) for r in range(budget) if mag[order[r]] > threshold]
    found = {}
    outs = locate_frequencies(cand, rounds, cfg, win) if cand else []
    located = [(bk, o) for bk, o in zip(cand, outs) if o is not None]
    if located:
        vals, ok = estimate_values([y0[bk] for bk, _ in located], [o.u for _, o in located], win)
        for (bk, o), v, good in zip(located, vals, ok):  # rank order
            if good:
                f = (base.sigma_inv * o.u) % n
                found[f] = found.get(f, 0j) + complex(v)
    for f in sorted(found):
        state.accumulated[f] = state.accumulated.get(f, 0j) + found[f]
    state.k_m = (state.k_m + 1) // 2
    state.b_m = state.b_m // 2 if state.b_m > 32 else state.b_m
    state.m += 1
    fs = sorted(found)
    return SparseSpectrum(n, np.array(fs, np.int64), np.array([found[f] for f in fs], np.complex128))
