"""Aggregate an ncu 'source' page (--print-source cuda,sass --csv) per CUDA
source line: warp-stall samples and executed warp instructions.
usage: ncu -i REP --page source --csv -k regex:K --print-source cuda,sass > x.csv
       python tools/ncu_lines.py x.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur_file = "?"
hdr = None
agg = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Line No":
        hdr = {k: i for i, k in enumerate(r)}
        continue
    if hdr is None or r[0] == "" or r[0] == "Function Name":
        continue
    try:
        samp = int(r[4] or 0)
        inst = int(r[7] or 0)
    except (ValueError, IndexError):
        continue
    agg.append((samp, inst, cur_file, r[0], r[1][:90]))
tot = sum(a[0] for a in agg) or 1
toti = sum(a[1] for a in agg) or 1
print(f"total samples {tot}, warp-instructions {toti}")
for s, i, f, ln, src in sorted(agg, reverse=True)[:top]:
    print(f"{100*s/tot:5.1f}% {100*i/toti:5.1f}%i {f}:{ln:>4} {src}")
