"""Aggregates an ncu --csv launch list (gpu__time_duration.sum) per kernel
name: count, total and mean time.  usage: python tools/ncu_agg.py file.csv [top]"""
import collections
import csv
import re
import sys

lines = [ln for ln in open(sys.argv[1]) if ln.startswith('"')]
rows = list(csv.reader(lines))
hdr = {k: i for i, k in enumerate(rows[0])}
tot = collections.defaultdict(lambda: [0, 0.0])
dram = collections.defaultdict(float)  # bytes, when the capture has dram__bytes_*
for r in rows[1:]:
    if len(r) < len(hdr):
        continue
    m = re.search(r"(\w+)(<[^(]*>)?\(", r[hdr["Kernel Name"]])
    name = m.group(1) if m else r[hdr["Kernel Name"]][:40]
    metric, unit = r[hdr["Metric Name"]], r[hdr["Metric Unit"]]
    v = float(r[hdr["Metric Value"]].replace(",", ""))
    if metric.startswith("dram__bytes"):
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6,
                 "GB": 1e9}.get(unit, 1)
        dram[name] += v * scale
        continue
    if metric != "gpu__time_duration.sum":
        continue
    us = v / 1000 if unit in ("ns", "nsecond") else v * 1000 if unit in ("ms", "msecond") else v
    tot[name][0] += 1
    tot[name][1] += us
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
total = sum(v[1] for v in tot.values())
print(f"{'kernel':34s} {'count':>6s} {'total ms':>10s} {'mean us':>9s} {'share':>6s} {'DRAM GB/s':>10s}")
for k, (c, us) in sorted(tot.items(), key=lambda t: -t[1][1])[:top]:
    bw = f"{dram[k] / (us * 1e-6) / 1e9:10.1f}" if k in dram else f"{'-':>10s}"
    print(f"{k:34s} {c:6d} {us / 1000:10.3f} {us / c:9.2f} {us / total:6.1%} {bw}")
print(f"{'all':34s} {sum(v[0] for v in tot.values()):6d} {total / 1000:10.3f}")
