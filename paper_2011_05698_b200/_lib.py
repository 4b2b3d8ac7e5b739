"""ctypes binding of include/msfft_b200.h (libmsfft_b200.so, built in-tree).

There is deliberately no fallback: if the CUDA library is missing or no GPU
is visible, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MSFFT_B200_LIB") or os.path.join(HERE, "libmsfft_b200.so")

MSFFT_OK, MSFFT_ERR_INVALID_ARGUMENT, MSFFT_ERR_DOMAIN, MSFFT_ERR_CUDA, MSFFT_ERR_RUNTIME = range(5)
MSFFT_C128, MSFFT_C64 = 0, 1
MSFFT_HOST, MSFFT_DEVICE = 0, 1
MSFFT_FLAG_ASSUME_VALID = 1
MSFFT_FLAG_STAGE_TIMES = 2
MSFFT_FLAG_SERIAL = 4
MSFFT_FLAG_ASYNC = 8
MAX_ITERATIONS = 64

# Every symbol include/msfft_b200.h declares.
EXPORTED = (
    "msfft_version", "msfft_device_count", "msfft_sfft4", "msfft_plan_create",
    "msfft_plan_destroy", "msfft_plan_stats", "msfft_execute", "msfft_plan_launches",
    "msfft_window", "msfft_window_response", "msfft_trace", "msfft_plan_stage_times",
    "msfft_plan_gather_traffic", "msfft_sigma_plan", "msfft_tau_plan",
    "msfft_plan_values_per_signal", "msfft_encode_values", "msfft_decode_values",
    "msfft_encode_values_part", "msfft_decode_folds",
    "msfft_plan_ingest_samples", "msfft_plan_copy_bytes", "msfft_validate_signal", "msfft_generate_test_signal", "msfft_synthesize",
    "msfft_add_awgn", "msfft_dft_dense", "msfft_idft_dense", "msfft_top_k_spectrum",
    "msfft_error_metrics", "msfft_signal_file_length", "msfft_read_signal_file",
    "msfft_write_signal_file", "msfft_write_truth_csv", "msfft_read_truth_csv",
    "msfft_phase_experiment", "msfft_plan_sync", "msfft_bucketize", "msfft_predict_buckets",
    "msfft_locate_frequency", "msfft_estimate_values", "msfft_mod_inverse", "msfft_bucket_of",
    "msfft_stage_count", "msfft_tau_schedule", "msfft_config_validate",
    "msfft_check_parameter_bounds", "msfft_initial_bucket_count", "msfft_phase_of",
    "msfft_position_phase", "msfft_circular_phase_distance", "msfft_locate_step",
    "msfft_bucketize_taps",
)

i64, u64, f64, i32, u32 = C.c_int64, C.c_uint64, C.c_double, C.c_int32, C.c_uint32
P = C.POINTER
VP = C.c_void_p


class Stats(C.Structure):
    _fields_ = [
        ("samples_used", i64),
        ("samples_round_sum", i64),
        ("sample_fraction", f64),
        ("runtime_ms", f64),
        ("iterations", i32),
        ("reserved", i32),
        ("b_first", i64),
        ("stage_counts", i32 * MAX_ITERATIONS),
    ]


class PhaseHistogramC(C.Structure):
    _fields_ = [("snr_db", f64), ("n", i64), ("k", i64), ("l_width", i64), ("trials", i64),
                ("bin_mass", f64 * 70), ("p50", f64), ("p99", f64), ("max", f64)]


class PhaseTrialC(C.Structure):
    _fields_ = [("dphi", f64), ("u", i64), ("bucket", i64), ("tau", i64), ("y0", f64 * 2),
                ("y_tau", f64 * 2), ("measured_phi", f64), ("true_phi", f64)]


class EvalMetricsC(C.Structure):
    _fields_ = [("l0_err", i64), ("l1_err", f64), ("l2_err", f64)]


_lib = None


def lib() -> C.CDLL:
    """Load (once) and return the CUDA library; raises if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2011_05698_b200.build` "
            "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    E = [C.c_char_p, C.c_size_t]
    L.msfft_version.restype = C.c_char_p
    L.msfft_device_count.restype = C.c_int
    L.msfft_sfft4.argtypes = [VP, i64, i32, i32, i64, i64, f64, u64, f64, i64, P(i64), P(f64),
                              P(i64), P(Stats)] + E
    L.msfft_plan_create.argtypes = [i64, i64, i64, f64, f64, i32, i32, P(VP)] + E
    L.msfft_plan_destroy.argtypes = [VP]
    L.msfft_plan_destroy.restype = None
    L.msfft_plan_stats.argtypes = [VP, P(Stats)]
    L.msfft_execute.argtypes = [VP, i64, VP, i64, i32, P(u64), VP, VP, VP, i32, u32, VP,
                                P(f64)] + E
    L.msfft_sigma_plan.argtypes = [u64, i64, i32, P(i64), P(i64)] + E
    L.msfft_sigma_plan.restype = C.c_int
    L.msfft_tau_plan.argtypes = [f64, i64, i64, f64, P(i64), i32, P(i32)] + E
    L.msfft_tau_plan.restype = C.c_int
    L.msfft_plan_gather_traffic.argtypes = [VP, i64, P(u64), P(i64), P(i64)]
    L.msfft_plan_gather_traffic.restype = C.c_int
    L.msfft_plan_stage_times.argtypes = [VP, P(f64)]
    L.msfft_plan_stage_times.restype = C.c_int
    L.msfft_plan_launches.argtypes = [VP, i64, u32]
    L.msfft_plan_launches.restype = i64
    # split-phase / ingest entry points (absent from diagnostic builds of
    # older sources, which tools/build_variant.py can produce)
    if hasattr(L, "msfft_plan_sync"):
        L.msfft_plan_sync.argtypes = [VP, VP] + E
        L.msfft_plan_sync.restype = C.c_int
    L.msfft_validate_signal.argtypes = [VP, i64, i64, i64, i64, i32, i32, VP, P(f64),
                                        C.c_char_p, C.c_size_t]
    L.msfft_validate_signal.restype = C.c_int
    L.msfft_plan_copy_bytes.argtypes = [VP, P(i64), P(i64)]
    L.msfft_plan_copy_bytes.restype = C.c_int
    if hasattr(L, "msfft_plan_ingest_samples"):
        L.msfft_plan_ingest_samples.argtypes = [VP]
        L.msfft_plan_ingest_samples.restype = i64
    if hasattr(L, "msfft_encode_values"):
        L.msfft_plan_values_per_signal.argtypes = [VP]
        L.msfft_plan_values_per_signal.restype = i64
        L.msfft_encode_values.argtypes = [VP, i64, VP, i64, i64, i64, P(u64), VP, u32, VP] + E
        L.msfft_encode_values.restype = C.c_int
        L.msfft_decode_values.argtypes = [VP, i64, VP, P(u64), VP, VP, VP, VP] + E
        L.msfft_encode_values_part.argtypes = [VP, i64, VP, i64, i64, i64, P(u64), VP, u32,
                                               VP] + E
        L.msfft_encode_values_part.restype = C.c_int
        L.msfft_decode_folds.argtypes = [VP, i64, VP, P(u64), VP, VP, VP, VP] + E
        L.msfft_decode_folds.restype = C.c_int
        L.msfft_decode_values.restype = C.c_int
    if hasattr(L, "msfft_generate_test_signal"):
        CP = C.c_char_p
        L.msfft_generate_test_signal.argtypes = [i64, i64, u64, i32, i32, VP, VP, VP,
                                                 P(i32)] + E
        L.msfft_synthesize.argtypes = [i64, VP, VP, i64, i32, i32, VP, P(i32)] + E
        L.msfft_add_awgn.argtypes = [VP, i64, i32, i32, f64, u64] + E
        L.msfft_dft_dense.argtypes = [VP, i64, i64, i32, i32, VP] + E
        L.msfft_idft_dense.argtypes = [VP, i64, i64, i32, VP] + E
        L.msfft_top_k_spectrum.argtypes = [VP, i64, i64, i32, VP, VP, P(i64)] + E
        L.msfft_error_metrics.argtypes = [i64, VP, VP, i64, i64, VP, VP, i64, i64,
                                          P(EvalMetricsC)] + E
        L.msfft_signal_file_length.argtypes = [CP, P(i64)] + E
        L.msfft_read_signal_file.argtypes = [CP, i32, i32, VP, i64, P(i64)] + E
        L.msfft_write_signal_file.argtypes = [CP, VP, i64, i32, i32] + E
        L.msfft_write_truth_csv.argtypes = [CP, VP, VP, i64] + E
        L.msfft_read_truth_csv.argtypes = [CP, i64, VP, VP, i64, P(i64)] + E
        if hasattr(L, "msfft_phase_experiment"):
            L.msfft_phase_experiment.argtypes = [i64, i64, i64, VP, i64, i64, u64,
                                                 P(PhaseHistogramC), P(PhaseTrialC)] + E
            L.msfft_phase_experiment.restype = C.c_int
        for fn in ("msfft_generate_test_signal", "msfft_synthesize", "msfft_add_awgn",
                   "msfft_dft_dense", "msfft_idft_dense", "msfft_top_k_spectrum",
                   "msfft_error_metrics", "msfft_signal_file_length", "msfft_read_signal_file",
                   "msfft_write_signal_file", "msfft_write_truth_csv", "msfft_read_truth_csv"):
            getattr(L, fn).restype = C.c_int
    if hasattr(L, "msfft_bucketize"):  # component API
        L.msfft_bucketize.argtypes = [VP, i64, i32, i32, i64, f64, VP, VP, i64, VP, i32,
                                      P(i64)] + E
        L.msfft_predict_buckets.argtypes = [i64, i64, f64, VP, VP, i64, VP, VP, i64, VP, i32] + E
        L.msfft_locate_frequency.argtypes = [i64, i64, i64, f64, VP, i64, VP, VP, i64, VP, VP,
                                             VP, i32] + E
        L.msfft_estimate_values.argtypes = [i64, i64, f64, VP, VP, i64, VP, VP, i32] + E
        for fn in ("msfft_bucketize", "msfft_predict_buckets", "msfft_locate_frequency",
                   "msfft_estimate_values"):
            getattr(L, fn).restype = C.c_int
    # scalar plan helpers (host) and the batched locate arithmetic (device)
    L.msfft_mod_inverse.argtypes = [i64, i64, P(i64)] + E
    L.msfft_bucket_of.argtypes = [i64, i64, i64]
    L.msfft_bucket_of.restype = i64
    L.msfft_stage_count.argtypes = [f64, i64, f64, P(i32)] + E
    L.msfft_tau_schedule.argtypes = [f64, i64, P(i64)] + E
    L.msfft_config_validate.argtypes = [i64, f64] + E
    L.msfft_check_parameter_bounds.argtypes = [f64, i64, f64, P(i32), P(f64)] + E
    L.msfft_initial_bucket_count.argtypes = [i64, i64, f64, P(i64)] + E
    L.msfft_phase_of.argtypes = [VP, i64, VP, VP] + E
    L.msfft_position_phase.argtypes = [VP, VP, i64, i64, VP] + E
    L.msfft_circular_phase_distance.argtypes = [VP, VP, i64, VP] + E
    L.msfft_locate_step.argtypes = [VP, VP, VP, i64, i64, f64, i64, VP] + E
    L.msfft_bucketize_taps.argtypes = [i64, i64, f64, VP, i64, VP, P(i64)] + E
    for fn in ("msfft_mod_inverse", "msfft_stage_count", "msfft_tau_schedule",
               "msfft_config_validate", "msfft_check_parameter_bounds",
               "msfft_initial_bucket_count", "msfft_phase_of", "msfft_position_phase",
               "msfft_circular_phase_distance", "msfft_locate_step", "msfft_bucketize_taps"):
        getattr(L, fn).restype = C.c_int
    L.msfft_window.argtypes = [i64, i64, f64, i32, P(i64), P(f64), i64] + E
    L.msfft_window_response.argtypes = [i64, i64, f64, i32, P(i64), i64, P(f64)] + E
    L.msfft_trace.argtypes = [VP, i64, i32, i64, i64, f64, u64, f64, P(f64), P(f64), P(i64),
                              P(i64), P(f64), i64, P(i64), P(f64), P(i64)] + E
    for fn in ("msfft_sfft4", "msfft_plan_create", "msfft_plan_stats", "msfft_execute",
               "msfft_window", "msfft_window_response", "msfft_trace"):
        getattr(L, fn).restype = C.c_int
    _lib = L
    return L
