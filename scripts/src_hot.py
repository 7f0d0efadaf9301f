"""Summarise an `ncu --page source --csv --print-source cuda,sass` dump:
per CUDA source line (and file), warp-instructions executed and stall samples."""
import csv
import sys
from collections import defaultdict

def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = None
cur_file = None
per = defaultdict(lambda: [0, 0, 0, ""])
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if len(r) > 3 and r[0] == "Line No":
        hdr = r
        ie = hdr.index("Instructions Executed")
        ss = hdr.index("Warp Stall Sampling (All Samples)")
        sn = hdr.index("Warp Stall Sampling (Not-issued Samples)")
        continue
    if hdr is None or len(r) < len(hdr) or r[0] == "":
        continue
    try:
        k = (cur_file, int(r[0]))
    except ValueError:
        continue
    p = per[k]
    p[0] += num(r[ie])
    p[1] += num(r[ss])
    p[2] += num(r[sn])
    p[3] = r[1][:90]
tot_i = sum(v[0] for v in per.values())
tot_s = sum(v[1] for v in per.values())
print(f"total warp-inst {tot_i:,}  stall samples {tot_s:,}")
for k, v in sorted(per.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{k[0]:>22}:{k[1]:<5} inst {100*v[0]/tot_i:5.1f}%  stall {100*v[1]/tot_s:5.1f}%  | {v[3]}")
