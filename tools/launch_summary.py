#!/usr/bin/env python
"""Summarise an ncu --csv launch list (gpu__time_duration.sum): per-kernel totals and the sequence."""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
tot, seq = {}, []
for r in rows[1:]:
    name = r[ki].split("(")[0].split("<")[0].replace("void ", "").replace("pfg::", "")
    v = float(r[vi].replace(",", ""))
    us = {"ns": v / 1e3, "us": v, "usecond": v, "ms": v * 1e3, "msecond": v * 1e3}.get(r[ui], v / 1e3)
    tot[name] = tot.get(name, 0.0) + us
    seq.append((name, round(us, 1)))
print("per kernel (us):", {k: round(v, 1) for k, v in tot.items()}, "sum %.1f" % sum(tot.values()))
print("sequence:", seq[:80])
