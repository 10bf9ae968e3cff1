#!/usr/bin/env python
"""Hot CUDA source lines from `ncu -i rep --page source --csv --print-source cuda,sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
res, fp, hdr = [], None, None
for r in rows:
    if r and r[0] == "File Path":
        fp = r[1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        try:
            samp = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
            inst = float(r[hdr.index("Instructions Executed")] or 0)
        except ValueError:
            continue
        res.append((samp, inst, fp.split("/")[-1], r[0], r[1].strip()[:100]))
tot = sum(x[0] for x in res) or 1
ti = sum(x[1] for x in res) or 1
print("total samples", tot, "warp instructions", ti)
for x in sorted(res, key=lambda t: -t[0])[:top]:
    print("%5.1f%% %5.1f%%  %s:%s  %s" % (100 * x[0] / tot, 100 * x[1] / ti, x[2], x[3], x[4]))
