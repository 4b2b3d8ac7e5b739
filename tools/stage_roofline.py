"""Per-stage roofline of one transform from an ncu launch list:

    ncu --clock-control none --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,\\
        dram__bytes_write.sum,sm__inst_executed_pipe_fp64.sum,\\
        sm__sass_thread_inst_executed_op_dadd_pred_on.sum,\\
        sm__sass_thread_inst_executed_op_dmul_pred_on.sum,\\
        sm__sass_thread_inst_executed_op_dfma_pred_on.sum,\\
        sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,\\
        smsp__issue_active.avg.pct_of_peak_sustained_active \\
        python tools/profile_c3.py --reps 2 > c3.csv
    python tools/stage_roofline.py c3.csv --workload "C3 ..." [--anchor encode_kernel]

The last execute (from its last `--anchor` launch on) is summarised per stage
(encode / bucket_fft / decode / other): time, DRAM bytes and GB/s against the
measured HBM peak, FP64 thread operations (DADD + DMUL + DFMA, non-FMA code
counts one op each) and their rate against the measured FP64 peak
(profiles/r02/fp64_peak.log: 1.855e13 DADD/DMUL thread-ops/s), the FP64-pipe
active fraction and issue-active fraction (duration-weighted).  Kernels run
back to back under ncu (no programmatic overlap): times are an upper bound."""
import argparse
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_05698_b200.provenance import csrc_sha256  # noqa: E402

HBM_PEAK = 6526.2        # GB/s, MEASURED_PEAKS.json hbm_gbs (copy)
FP64_PEAK = 1.8552e13    # DADD thread-ops/s, tools/fp64_peak.cu on this pool


def stage_of(name):
    if name.startswith(("encode_kernel", "fused_kernel")):
        return "encode"
    if name.startswith(("fft_smem", "stages_kernel", "stages_sets_kernel", "bitrev_inplace")):
        return "bucket_fft"
    if name.startswith(("sigma_kernel", "validate_kernel", "zero_words", "compact_gather")):
        return "other"
    if name.startswith(TORCH):  # the caller's own tensor ops (e.g. run_c5's x * 2)
        return None
    return "decode"


TORCH = ("StoreWithoutCast", "elementwise", "vectorized", "direct_copy", "unrolled_elementwise")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--workload", default="")
    ap.add_argument("--anchor", default="encode_kernel")
    ap.add_argument("--anchor-grid-max", action="store_true",
                    help="anchor at the last --anchor launch with the largest grid (the serial "
                         "execute's single encode, not the overlapped path's per-group encodes) "
                         "and stop at the next --anchor launch")
    a = ap.parse_args()
    lines = open(a.csv).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(lines[start:]))
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    gi = h.index("Grid Size")
    launches = {}
    for r in rows[1:]:
        d = launches.setdefault(int(r[ii]), {"name": r[ki].split("(")[0].split("::")[-1].split("<")[0],
                                             "grid": r[gi]})
        try:
            d[r[mi]] = float(r[vi].replace(",", ""))
        except ValueError:
            pass
    seq = [launches[i] for i in sorted(launches)]
    starts = [i for i, d in enumerate(seq) if d["name"] == a.anchor]
    last = seq[starts[-1]:]
    if a.anchor_grid_max:
        gsize = lambda d: eval(d["grid"].replace("(", "").replace(")", "").replace(", ", "*"))  # noqa: E731
        big = max(gsize(seq[i]) for i in starts)
        i0 = [i for i in starts if gsize(seq[i]) == big][-1]
        nxt = [i for i in starts if i > i0]
        last = seq[i0:nxt[0] if nxt else len(seq)]
    out, kern = {}, {}
    for d in last:
        us = d.get("gpu__time_duration.sum", 0.0) / 1e3
        ops = sum(d.get(f"sm__sass_thread_inst_executed_op_{o}_pred_on.sum", 0.0)
                  for o in ("dadd", "dmul", "dfma"))
        if stage_of(d["name"]) is None:
            continue
        for key, table in ((stage_of(d["name"]), out), (d["name"], kern)):
            st = table.setdefault(key, {"launches": 0, "us": 0.0, "dram_bytes": 0.0,
                                        "fp64_thread_ops": 0.0, "fp64_warp_inst": 0.0,
                                        "_pipe": 0.0, "_issue": 0.0})
            st["launches"] += 1
            st["us"] += us
            st["dram_bytes"] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
            st["fp64_thread_ops"] += ops
            st["fp64_warp_inst"] += d.get("sm__inst_executed_pipe_fp64.sum", 0.0)
            st["_pipe"] += us * d.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 0.0)
            st["_issue"] += us * d.get("smsp__issue_active.avg.pct_of_peak_sustained_active", 0.0)
    for table in (out, kern):
        for st in table.values():
            t = st["us"] * 1e-6
            st["dram_gbs"] = st["dram_bytes"] / t / 1e9 if t else 0.0
            st["hbm_frac"] = st["dram_gbs"] / HBM_PEAK
            st["fp64_ops_per_s"] = st["fp64_thread_ops"] / t if t else 0.0
            st["fp64_frac_of_measured_peak"] = st["fp64_ops_per_s"] / FP64_PEAK
            st["fp64_pipe_active_frac"] = st.pop("_pipe") / st["us"] / 100.0 if st["us"] else 0.0
            st["issue_active_frac"] = st.pop("_issue") / st["us"] / 100.0 if st["us"] else 0.0
    res = {"workload": a.workload, "source": os.path.basename(a.csv),
           "peaks": {"hbm_gbs": HBM_PEAK, "fp64_thread_ops_per_s": FP64_PEAK,
                     "fp64_source": "profiles/r02/fp64_peak.log (DADD/DMUL, 8 chains/thread)"},
           "note": "ncu launch list, last execute, kernels serialised (upper bound of live time)",
           "csrc_sha256": csrc_sha256(),
           "stages": out,
           "kernels": dict(sorted(kern.items(), key=lambda kv: -kv[1]["us"]))}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
