"""Key counters of one kernel launch from an ncu report:

    python tools/ncu_summary.py report.ncu-rep [--workload TEXT] [--traffic out.json
                                [--batch B --n N]]

Reads `ncu -i report --page raw --csv` (first launch in the report) and prints a
JSON summary: duration, DRAM bytes, occupancy, issue activity, FP64 pipe,
and the share of each warp-stall reason.  --traffic also writes the
DRAM-bytes record bench.py reads for roofline.traffic (bench.py uses it only
when its batch and n match the run, so pass --batch and --n)."""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_05698_b200.provenance import csrc_sha256  # noqa: E402

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "launch__registers_per_thread": "registers",
    "launch__shared_mem_per_block_dynamic": "smem_dynamic",
    "launch__occupancy_limit_shared_mem": "occupancy_limit_smem",
    "launch__occupancy_limit_registers": "occupancy_limit_regs",
    "smsp__inst_executed.sum": "warp_instructions",
}
STALL_PREFIX2 = "smsp__pcsamp_warps_issue_stalled_"


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], check=True,
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    header = rows[0]
    units = rows[1]
    return header, units, rows[2:]


def to_float(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def summarize(rep, kernel=None):
    import re
    header, units, data = raw_rows(rep)
    col = {h: i for i, h in enumerate(header)}
    row = data[0]
    if kernel:
        row = next(r for r in data if re.search(kernel, r[col["Kernel Name"]]))
    s = {"kernel": row[col["Kernel Name"]] if "Kernel Name" in col else None}
    for metric, name in KEYS.items():
        if metric in col:
            s[name] = to_float(row[col[metric]])
            s[name + "_unit"] = units[col[metric]]
    stalls = {}
    for h, i in col.items():
        if h.startswith(STALL_PREFIX2) and not h.endswith("not_issued"):
            reason = h[len(STALL_PREFIX2):]
            v = to_float(row[i])
            if v is not None:
                stalls[reason] = v
    total = sum(stalls.values())
    if total > 0:
        s["stall_share"] = {k: round(v / total, 4)
                            for k, v in sorted(stalls.items(), key=lambda kv: -kv[1]) if v > 0}
    return s


def scaled_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return None if v is None else v * scale


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--workload", default="")
    ap.add_argument("--traffic")
    ap.add_argument("--batch", type=int)
    ap.add_argument("--n", type=int)
    ap.add_argument("--kernel", help="regex: summarise the first launch whose name matches")
    a = ap.parse_args()
    s = summarize(a.report, a.kernel)
    if a.workload:
        s["workload"] = a.workload
    # the native sources the capture ran on (run this on the same tree)
    s["csrc_sha256"] = csrc_sha256()
    print(json.dumps(s, indent=1))
    if a.traffic:
        rd = scaled_bytes(s.get("dram_read"), s.get("dram_read_unit"))
        wr = scaled_bytes(s.get("dram_write"), s.get("dram_write_unit"))
        dur = s.get("duration")
        dur_ms = dur / 1e6 if s.get("duration_unit") == "nsecond" else (
            dur / 1e3 if s.get("duration_unit") == "usecond" else dur)
        if a.batch is None or a.n is None:
            raise SystemExit("--traffic needs --batch and --n (bench.py matches them)")
        rec = {"kernel": s["kernel"], "batch": a.batch, "n": a.n,
               "dram_bytes_per_launch": int(rd + wr),
               "dram_bytes_read": int(rd), "dram_bytes_write": int(wr),
               "duration_ms_under_ncu": dur_ms, "csrc_sha256": s["csrc_sha256"],
               "source": f"{a.report} (ncu --set full --clock-control none)"}
        with open(a.traffic, "w") as f:
            json.dump(rec, f, indent=1)
