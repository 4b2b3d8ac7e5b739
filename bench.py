#!/usr/bin/env python
"""Headline benchmark: batched sFFT4.0 throughput (BASELINE.json metric).

Workload (BASELINE.json configs[3], "C4"): independent signals, each N=2^22,
K=64, complex64, unit-magnitude tones with uniform phases, AWGN at 25 dB,
per-signal seeds; delta = 1e-6 (noisy), l = 16, q = 1 (the reference bench's
rules, proj/src/bench.cpp:124, bench.hpp:40-41).  A "step" is one sfft4 of
the whole batch (1024 signals per GPU; weak scaling under torchrun).

  python bench.py [--gpus N --steps K --warmup W]            # this framework
  python bench.py --impl reference [...]                     # reference CPU arm

The b200 arm prints one JSON line with:
  value     transforms/s, device-resident inputs, device-timed (CUDA events on
            the execution stream), max over ranks; every step is a full
            validating sfft4 (finiteness scan of every sample, as the
            reference's sfft4.cpp:133 does per call); value_assume_valid is
            the same steps with MSFFT_FLAG_ASSUME_VALID
  e2e       the same metric through the public API with pinned HOST inputs:
            every step ingests the batch (sparse ingest: the samples the
            transform reads, gathered by host threads; finiteness scan of
            every sample) host->device and copies the sparse results
            device->host inside the timed region
  roofline  the validating step's one kernel (fused_val_kernel: finiteness
            scan + gather/fold/FFT + decode): algorithmic bytes = every byte
            of x once / its CUDA-event time; roofline_gather: the
            ASSUME_VALID fused kernel, algorithmic bytes = the distinct 32-B
            sectors the gather loads (from the plan); roofline_validate: the
            standalone finiteness scan kernel (n * 8 bytes per signal)
  cpu_baseline  the reference's own CPU code (oracle/_ref, compiled from
            /root/reference) on a bounded sample, all host threads
The reference arm (--impl reference) times that same CPU code alone.
Inputs (32 GiB per GPU) are far larger than L2 (126 MB): no flush needed.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "sparse transforms/sec (N=2^22,K=64 batch) + filter gather HBM GB/s vs peak"
SIG_BASE = 0xC4C4_0000


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--batch", type=int, default=1024)
    ap.add_argument("--log2n", type=int, default=22)
    ap.add_argument("--k", type=int, default=64)
    ap.add_argument("--snr", type=float, default=25.0)
    ap.add_argument("--e2e-steps", type=int, default=4)
    ap.add_argument("--e2e-warmup", type=int, default=6,
                    help="untimed host-path calls first (staging buffers, the adaptive "
                         "host-scan / DMA validation split)")
    ap.add_argument("--cpu-sample", type=int, default=0,
                    help="signals per CPU step (default: 2 per host thread)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-clocks", action="store_true", help="diagnostics: no nvidia-smi sampler")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: --batch signals per GPU; strong: --batch signals in total")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def load_peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.lines: list[str] = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.device)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax),
                "reasons": sorted(reasons), "samples": len(sm)}


def e2e_batch(batch: int, sig_bytes: int, local_ranks: int) -> int:
    """Signals per rank for the e2e leg: all of them when the host can pin
    them (half of the available memory split over the local ranks), else as
    many as fit (at least 8)."""
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:  # noqa: BLE001
        return batch
    fit = int(avail * 0.5 / max(local_ranks, 1) / sig_bytes)
    return max(min(batch, fit), min(batch, 8))


def current_csrc():
    from paper_2011_05698_b200.provenance import csrc_sha256
    return csrc_sha256()


def profile_record(name, csrc):
    """A committed ncu summary under profiles/, or None unless it carries
    the content hash of the native sources this run was built from."""
    path = os.path.join(REPO, "profiles", name)
    if not os.path.exists(path):
        return None
    with open(path) as f:
        d = json.load(f)
    if d.get("csrc_sha256") != csrc:
        return None
    return d


def pipe_evidence(csrc):
    """FP64-pipe and SM utilisation of the fused launch and of the decode
    (the FFT / locate / estimate stages) from committed ncu captures of the
    same workload on the same native sources, or None."""
    out = {}
    for key, name in (("fused_val_kernel", "fused_val_ncu_summary.json"),
                      ("fused_kernel", "fused_ncu_summary.json"),
                      ("decode_kernel", "decode_c4_ncu_summary.json"),
                      ("validate_kernel", "validate_ncu_summary.json")):
        d = profile_record(name, csrc)
        if d is None:
            continue
        def num(raw, short):  # raw ncu metric names or tools/ncu_summary.py keys
            v = d.get(raw, d.get(short))
            try:
                return float(v) / 100.0
            except (TypeError, ValueError):
                return None
        out[key] = {"fp64_pipe_frac": num("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
                                          "fp64_pipe_pct"),
                    "issue_active_frac": num("smsp__issue_active.avg.pct_of_peak_sustained_active",
                                             "issue_active_pct"),
                    "sm_throughput_frac": num("sm__throughput.avg.pct_of_peak_sustained_elapsed",
                                              "sm_throughput_pct"),
                    "top_stalls": d.get("stall_share"), "source": f"profiles/{name}"}
    return out or None


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_oracle():
    """The reference's own CPU implementation (compiled from /root/reference
    into oracle/_ref), else the restatement (oracle/_port)."""
    from oracle import available, load
    if available("reference"):
        return load("reference"), "reference"
    return load("port"), "port"


def prewarm_reference_windows(orc, n, k, delta):
    """Design the reference's windows (its own code, its own cache) in
    parallel threads; untimed, as the reference resolves them before its
    timer (proj/src/sfft4.cpp:146-154)."""
    b = orc.initial_bucket_count(n, k, delta)
    bs = []
    for _ in range(int(math.ceil(math.log2(k))) + 2):
        bs.append(b)
        b = b // 2 if b > 32 else b
    ts = [threading.Thread(target=orc.window, args=(n, bb, delta, False)) for bb in sorted(set(bs))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()


def cpu_sample_signals(x_dev_or_host, count):
    import torch
    xs = x_dev_or_host[:count]
    if isinstance(xs, torch.Tensor):
        xs = xs.cpu().numpy()
    return np.ascontiguousarray(xs.astype(np.complex64))


def run_cpu(orc, xs, k, aseeds, delta, threads, steps, warmup):
    """Times the reference sfft4 over `xs` (one step = all of xs) on `threads`
    host threads; returns (transforms/s, per-step results of the last step)."""
    for _ in range(warmup):
        orc.sfft4_batch_c64(xs, k, 16, 1.0, aseeds, delta, threads)
    t0 = time.perf_counter()
    res = None
    for _ in range(steps):
        res, _wall = orc.sfft4_batch_c64(xs, k, 16, 1.0, aseeds, delta, threads)
    dt = time.perf_counter() - t0
    return steps * len(xs) / dt, res


def main():
    args = parse()
    rank, world, local = dist_env()
    n, k, delta = 1 << args.log2n, args.k, 1e-6
    config = {"workload": f"C4: batch of N=2^{args.log2n}, K={k}, complex64, |c|=1, "
                          f"AWGN {args.snr:g} dB, per-signal seeds (BASELINE.json configs[3])",
              "n": n, "k": k, "l": 16, "q": 1.0, "delta": delta, "per_gpu_batch": args.batch if args.scaling == "weak" else
              -(-args.batch // world), "global_batch": args.batch * world
              if args.scaling == "weak" else args.batch, "snr_db": args.snr,
              "parallelism": f"signal-sharded x{world} (no collective on the data path)",
              "l2_policy": "inputs (32 GiB/GPU) >> L2 (126 MB); no flush",
              "input_dtype": "complex64 (upcast exactly; all arithmetic in float64)"}

    if args.impl == "reference":
        return run_reference_arm(args, rank, world, n, k, delta, config)

    import torch
    import paper_2011_05698_b200 as M
    from paper_2011_05698_b200.workloads import algo_seed, make_batch, signal_seed

    # one GPU per local rank; the modulo only matters for the functional
    # multi-rank check on a one-GPU box (tools/bench_ranks_check.sh), whose
    # ranks share the device and use gloo (MSFFT_BENCH_DIST_BACKEND)
    gpu = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("MSFFT_BENCH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    from paper_2011_05698_b200.dist import max_over_ranks, rank_seeds, sum_over_ranks
    seeds = rank_seeds(SIG_BASE, args.batch, rank, world, args.scaling)
    aseeds = np.array([algo_seed(s) for s in seeds], dtype=np.uint64)
    x, _ = make_batch(n, k, seeds, args.snr, dev, "complex64")
    torch.cuda.synchronize()

    plan = M.Plan(n, k, M.MultiscaleConfig(16, 1.0), delta, "complex64", gpu)
    B = len(seeds)  # this rank's signals
    total = sum_over_ranks(B, dev) if world > 1 else B
    out_f = torch.empty((B, k), dtype=torch.int64, device=dev)
    out_c = torch.empty((B, k), dtype=torch.complex128, device=dev)
    out_n = torch.empty((B,), dtype=torch.int64, device=dev)
    out = (out_f, out_c, out_n)
    stream = torch.cuda.current_stream(dev)
    sh = stream.cuda_stream

    # Every timed step is a full sfft4 call as the reference defines it:
    # ComplexSignal::validate scans all n samples of every signal
    # (sfft4.cpp:133) before the transform.  The same steps with
    # ASSUME_VALID (a caller that validated at ingest) are timed after, as
    # value_assume_valid.
    seed_sets = (aseeds, aseeds ^ np.uint64(0x9E3779B97F4A7C15))
    plan.execute(x, aseeds, out=out, assume_valid=False, stream=sh)
    for i in range(args.warmup):
        plan.execute(x, seed_sets[i & 1], out=out, assume_valid=False, stream=sh)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(gpu)
    if not args.no_clocks:
        clocks.start()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)

    def timed(assume_valid):
        # the K steps are enqueued back to back (MSFFT_FLAG_ASYNC: no host
        # round trip between steps); two seed sets alternate so every step
        # uploads its seeds and recomputes the sigma plan; errors of the loop
        # (a non-finite sample, a decode failure) surface in sync()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for i in range(args.steps):
            plan.execute(x, seed_sets[i & 1], out=out, assume_valid=assume_valid, stream=sh,
                         async_=True)
        ev1.record(stream)
        torch.cuda.synchronize()
        plan.sync(sh)
        if world > 1:
            torch.distributed.barrier()
        t = ev0.elapsed_time(ev1) / args.steps
        return max_over_ranks(t, dev) if world > 1 else t

    ms = timed(False)
    for i in range(args.warmup):
        plan.execute(x, seed_sets[i & 1], out=out, assume_valid=True, stream=sh)
    ms_av = timed(True)
    clk = clocks.stop()
    value = total / (ms / 1e3)
    value_av = total / (ms_av / 1e3)

    # live time of the validation scan alone (ComplexSignal::validate over
    # the rank's batch), CUDA events around the kernel on the same stream
    val_ms = [M.validate_signal(x, stream=sh) for _ in range(3)]
    val_avg = sum(val_ms) / len(val_ms)
    val_bytes = B * n * 8

    # live per-launch time of the validating step's kernel (fused_val_kernel:
    # scan + encode + decode in one launch), CUDA events around each launch on
    # its stream; its algorithmic bytes are every byte of x once (the scan
    # reads all of them; the gathers read lines the scan also reads)
    vmain_ms = []
    for _ in range(max(3, min(args.steps, 10))):
        plan.execute(x, aseeds, out=out, assume_valid=False, stream=sh, stage_times=True)
        vmain_ms.append(plan.stage_times()[0])
    vmain_avg = sum(vmain_ms) / len(vmain_ms)
    val_fused = plan.launches(B, assume_valid=False) == 2

    # live per-launch time of the ASSUME_VALID kernel (fused encode+decode), CUDA
    # events around each launch on its stream
    main_ms = []
    for _ in range(max(3, min(args.steps, 10))):
        plan.execute(x, aseeds, out=out, assume_valid=True, stream=sh, stage_times=True)
        main_ms.append(plan.stage_times()[0])

    # roofline of the dominant kernel: the persistent fused encode+decode
    # launch (all of a step's device time but the sigma plan); its HBM work
    # is the gather, whose algorithmic bytes are the distinct 32-B sectors.
    loads, sectors = plan.gather_traffic(aseeds)
    alg_bytes = sectors * 32
    main_avg = sum(main_ms) / len(main_ms)
    achieved = alg_bytes / (main_avg / 1e3) / 1e9
    peak, peak_src = load_peaks()
    # diagnostic pass: encode and decode as separate launches
    enc_ms, dec_ms = [], []
    for _ in range(3):
        plan.execute(x, aseeds, out=out, assume_valid=True, stream=sh, stage_times=True,
                     serial=True)
        st = plan.stage_times()
        enc_ms.append(st[0])
        dec_ms.append(st[2])
    enc_avg = sum(enc_ms) / len(enc_ms)
    dec_avg = sum(dec_ms) / len(dec_ms)
    csrc = current_csrc()

    def ncu_traffic(name):
        """DRAM bytes per launch from a committed `ncu --set full` capture of
        the same workload on the same native sources (profiles/<name>), or None."""
        tj = profile_record(name, csrc)
        if tj is not None and tj.get("batch") == B and tj.get("n") == n:
            return tj.get("dram_bytes_per_launch")
        return None

    traffic = ncu_traffic("fused_traffic.json")
    vtraffic = ncu_traffic("fused_val_traffic.json")
    enc_traffic = ncu_traffic("encode_traffic.json")
    val_traffic = ncu_traffic("validate_traffic.json")

    # e2e through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e and args.e2e_steps > 0:
        # every rank pins a host copy of its signals: size it to the host
        # memory actually available (all local ranks share the host)
        be = e2e_batch(B, n * 8, int(os.environ.get("LOCAL_WORLD_SIZE", world)))
        xh = torch.empty((be, n), dtype=torch.complex64, pin_memory=True)
        xh.copy_(x[:be])
        eseeds = aseeds[:be]
        for _ in range(max(1, args.e2e_warmup)):
            plan.execute(xh, eseeds)  # warm the host path
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        h2d = d2h = 0
        for _ in range(args.e2e_steps):
            fh, ch, nh, _ = plan.execute(xh, eseeds)  # validating call, D2H results
            hb, db = plan.copy_bytes()
            h2d += hb
            d2h += db
        et = (time.perf_counter() - t0) / args.e2e_steps
        if world > 1:
            et = max_over_ranks(et, dev)
        etotal = sum_over_ranks(be, dev) if world > 1 else be
        ingest = plan.ingest_samples_per_signal
        e2e = {"value": etotal / et, "unit": "transforms/s", "signals_per_step": int(etotal),
               "h2d_bytes_per_step": int(sum_over_ranks(h2d, dev) if world > 1 else h2d)
               // args.e2e_steps,
               "ingest": (f"sparse: host threads gather the {ingest} samples per signal the "
                          "transform reads into pinned staging; the finiteness scan of all n "
                          "samples is split between host threads and whole rows the copy "
                          "engine moves for a device scan (both counted in h2d bytes)"
                          if ingest else "dense: whole signals copied"),
               "d2h_bytes_per_step": int(sum_over_ranks(d2h, dev) if world > 1 else d2h)
               // args.e2e_steps,
               "bytes_source": "counted by the library per call (msfft_plan_copy_bytes)",
               "ms_per_step": et * 1e3, "timing": "wall clock around msfft_execute (blocking)"}
        del xh

    # CPU baseline: the reference's own code on a bounded sample of the same bytes
    cpu = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu:
        orc, kind = reference_oracle()
        threads = os.cpu_count() or 1
        S = min(args.cpu_sample or max(8, min(2 * threads, 256)), B)
        prewarm_reference_windows(orc, n, k, delta)
        xs = cpu_sample_signals(x, S)
        rate, res = run_cpu(orc, xs, k, aseeds[:S], delta, threads, steps=1, warmup=0)
        cpu = {"value": rate, "unit": "transforms/s", "cores": threads, "kind": kind,
               "sample": f"{S} of the {B} batch signals (same bytes, c64 upcast to c128), "
                         f"one pass, {threads} std::thread workers, windows pre-designed",
               "cpu_model": cpu_model()}
        # parity of the GPU outputs on the sampled signals
        gf = out_f[:S].cpu().numpy()
        gc = out_c[:S].cpu().numpy()
        gn = out_n[:S].cpu().numpy()
        same = 0
        worst = 0.0
        for i in range(S):
            rf, rc = res[i].f, res[i].c
            m = int(gn[i])
            if m == len(rf) and np.array_equal(gf[i, :m], rf):
                same += 1
                floor = 10 * k * delta * float(np.max(np.abs(rc))) if m else 1.0
                err = np.max(np.abs(gc[i, :m] - rc) / np.maximum(np.abs(rc), floor)) if m else 0
                worst = max(worst, float(err))
        parity = {"signals": S, "support_identical": same, "max_rel_coef_err": worst,
                  "tolerance": 1e-4}

    launches = plan.launches(B, assume_valid=False) * args.steps
    line = {
        "metric": METRIC, "value": value, "unit": "transforms/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "step": "one validating sfft4 over the batch: ComplexSignal::validate scan of every "
                "sample (sfft4.cpp:133) + the transform, as the reference does per call",
        "value_assume_valid": value_av, "ms_per_step_assume_valid": ms_av,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded K-sparse spectra + AWGN, BASELINE.json configs[3] law)",
        "config": config,
        "roofline": ({"bound": "hbm",
                      "kernel": "fused_val_kernel (persistent: finiteness scan of every sample + "
                                "gather/window/fold/FFT + decode, one launch per validating step)",
                      "achieved": val_bytes / (vmain_avg / 1e3) / 1e9, "peak": peak,
                      "unit": "GB/s", "frac": val_bytes / (vmain_avg / 1e3) / 1e9 / peak,
                      "traffic": vtraffic, "peak_source": peak_src,
                      "algorithmic_bytes_per_launch": val_bytes,
                      "algorithmic_bytes": "every byte of x once (B * n * 8): the scan reads "
                                           "all samples, the gather's 8-B reads fall in the "
                                           "same lines (fetched ~4 chunks ahead of the scan, "
                                           "which then hits them in L2)",
                      "launch_ms": vmain_avg, "share_of_step": vmain_avg / ms,
                      "survey_8d_gather_metric": "roofline_gather: SURVEY 8(d) defines the "
                                                 "filter-gather roofline on the distinct 32-B "
                                                 "sectors of a transform that does not validate "
                                                 "(the ASSUME_VALID kernel); this kernel also "
                                                 "reads every sample for the finiteness scan, "
                                                 "so its algorithmic bytes are all of x",
                      "gather_sector_bytes_per_launch": alg_bytes,
                      "csrc_sha256": csrc} if val_fused else None),
        "roofline_gather": {"bound": "hbm",
                     "kernel": "fused_kernel (persistent: gather/window/fold/FFT + decode; "
                               "the ASSUME_VALID step)",
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": alg_bytes, "loads_per_launch": loads,
                     "launch_ms": main_avg, "share_of_step": main_avg / ms,
                     "note": "every random 8-B sample load fills a 128-B HBM line on B200, so "
                             "the 32-B-sector metric tops out at 0.25 of peak "
                             "(profiles/r01/gather_probe_*.log)",
                     "encode_only": {"kernel": "encode_kernel", "launch_ms": enc_avg,
                                     "achieved": alg_bytes / (enc_avg / 1e3) / 1e9,
                                     "frac": alg_bytes / (enc_avg / 1e3) / 1e9 / peak,
                                     "traffic": enc_traffic},
                     "decode_only_ms": dec_avg,
                     "pipes": pipe_evidence(csrc), "csrc_sha256": csrc},
        "roofline_validate": {"bound": "hbm", "kernel": "validate_kernel (finiteness scan)",
                              "achieved": val_bytes / (val_avg / 1e3) / 1e9, "peak": peak,
                              "unit": "GB/s",
                              "frac": val_bytes / (val_avg / 1e3) / 1e9 / peak,
                              "traffic": val_traffic, "algorithmic_bytes_per_launch": val_bytes,
                              "launch_ms": val_avg,
                              "share_of_step": val_avg / ms},
        "e2e": e2e, "cpu_baseline": cpu, "parity_sample": parity, "clocks": clk,
        "gpu_launches": launches,
    }
    if line["roofline"] is None:  # MSFFT_VAL_FUSED=0: separate scan + fused launch
        line["roofline"] = line["roofline_gather"]
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def run_reference_arm(args, rank, world, n, k, delta, config):
    """The reference's own CPU implementation on this box's host cores, same
    config/metric; rank 0 only under torchrun."""
    if rank != 0:
        return
    import torch
    from paper_2011_05698_b200.workloads import algo_seed, make_batch, signal_seed
    orc, kind = reference_oracle()
    threads = os.cpu_count() or 1
    S = args.cpu_sample or max(8, min(2 * threads, 256))
    dev = torch.device("cuda", 0) if torch.cuda.is_available() else torch.device("cpu")
    seeds = [signal_seed(SIG_BASE, i) for i in range(S)]
    aseeds = np.array([algo_seed(s) for s in seeds], dtype=np.uint64)
    x, _ = make_batch(n, k, seeds, args.snr, dev, "complex64")
    xs = cpu_sample_signals(x, S)
    prewarm_reference_windows(orc, n, k, delta)
    rate, _ = run_cpu(orc, xs, k, aseeds, delta, threads, steps=args.steps,
                      warmup=min(args.warmup, 1))
    line = {
        "metric": METRIC, "value": rate, "unit": "transforms/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": S / rate * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (same generator as the b200 arm)", "config": config,
        "impl": "reference",
        "cpu_baseline": {"value": rate, "unit": "transforms/s", "cores": threads, "kind": kind,
                         "sample": f"{S} signals per step, {threads} std::thread workers",
                         "cpu_model": cpu_model()},
        "e2e": {"value": rate, "unit": "transforms/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
