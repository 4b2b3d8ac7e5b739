"""Per-stage time and DRAM traffic of one C3 transform from an ncu launch
list (see profiles/README.md):

    ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,\\
        dram__bytes_write.sum --csv python tools/profile_c3.py --reps 2 > c3.csv
    python tools/c3_stages.py c3.csv [live_stage_ms_json]

Each serial execute has one encode_kernel launch; the last execute (from its
encode on) is summarised.
Kernels run back to back under ncu (no programmatic overlap), so the sum is
an upper bound of the live time."""
import csv
import json
import sys

PEAK = 6553.3  # GB/s, measured copy peak (MEASURED_PEAKS.json on the pool)


def stage_of(name):
    if name.startswith("encode_kernel"):
        return "encode"
    if name.startswith(("fft_smem", "stages_kernel", "bitrev_inplace")):
        return "bucket_fft"
    if name.startswith(("sigma_kernel", "validate_kernel")):
        return "other"
    return "decode"


lines = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.reader(lines[start:]))
h = rows[0]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
launches = {}
for r in rows[1:]:
    d = launches.setdefault(int(r[ii]), {"name": r[ki].split("(")[0].split("::")[-1].split("<")[0]})
    d[r[mi]] = float(r[vi].replace(",", ""))
seq = [launches[i] for i in sorted(launches)]
starts = [i for i, d in enumerate(seq) if d["name"] == "encode_kernel"]
last = seq[starts[-1]:]
out = {}
for d in last:
    st = out.setdefault(stage_of(d["name"]), {"launches": 0, "us": 0.0, "dram_bytes": 0.0})
    st["launches"] += 1
    st["us"] += d.get("gpu__time_duration.sum", 0.0) / 1e3
    st["dram_bytes"] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
for st in out.values():
    st["dram_gbs"] = st["dram_bytes"] / (st["us"] * 1e3) if st["us"] else 0.0
    st["frac_of_hbm_peak"] = st["dram_gbs"] / PEAK
res = {"workload": "C3: N=2^24, K=1000, c128, min-separated support, 30 dB (tools/profile_c3.py); "
                   "ncu launch list, last execute (serial path)",
       "peak_hbm_gbs": PEAK, "stages_under_ncu": out}
if len(sys.argv) > 2:
    res["live_stage_ms"] = json.load(open(sys.argv[2]))
print(json.dumps(res, indent=1))
