#!/usr/bin/env python
"""DRAM traffic per k_sims launch from an ncu CSV of one search (all its k_sims launches):
  ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --kernel-name regex:k_sims --csv --log-file X.csv python tools/prof_search.py --config 2
  python tools/ksims_traffic.py X.csv profiles/ksims_traffic_config2.json"""
import csv
import json
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi, ui, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("ID")
per = {}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3}
for r in rows[1:]:
    if "k_sims" not in r[ki]:
        continue
    d = per.setdefault(r[ii], {})
    d[r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
launches = list(per.values())
dram = [l["dram__bytes_read.sum"] + l["dram__bytes_write.sum"] for l in launches]
out = {"source": sys.argv[1].split("/")[-1] + " (ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum, one search, "
                                            "serialised, cold L2)",
       "launches": len(launches), "dram_bytes_per_launch": sum(dram) / len(dram),
       "dram_bytes_each": dram, "duration_s_each": [l["gpu__time_duration.sum"] for l in launches]}
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out))
