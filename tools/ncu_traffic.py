#!/usr/bin/env python
"""DRAM traffic of the query phase of one search (all kernels after the query preparation), from an
ncu launch list with dram__bytes_{read,write}.sum; writes profiles/query_phase_traffic_config<N>.json.

  ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none --csv --log-file gpurun_out/traffic.csv python tools/prof_search.py --config 2
  python tools/ncu_traffic.py gpurun_out/traffic.csv 2
"""
import csv
import json
import os
import sys

PREP = ("k_normalize", "k_hp_bits", "k_fht_qcodes", "k_qbounds")  # query preparation (first qbounds only)
src, cfg = sys.argv[1], int(sys.argv[2])
rows = [r for r in csv.reader(open(src)) if len(r) > 10]
h = rows[0]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3}
launches, cur = [], None
for r in rows[1:]:
    name = r[ki].split("(")[0].split("<")[0].replace("void ", "").replace("pfg::", "")
    key = (r[0], name)
    if cur is None or cur["key"] != key:
        cur = {"key": key, "name": name}
        launches.append(cur)
    cur[r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
seen_prep, q_bytes, q_time, per = set(), 0.0, 0.0, {}
for l in launches:
    n = l["name"]
    pk = next((x for x in PREP if n.startswith(x)), None)
    if pk and pk not in seen_prep:
        seen_prep.add(pk)
        continue
    b = l.get("dram__bytes_read.sum", 0) + l.get("dram__bytes_write.sum", 0)
    q_bytes += b
    q_time += l.get("gpu__time_duration.sum", 0)
    p = per.setdefault(n, [0.0, 0.0, 0])
    p[0] += b; p[1] += l.get("gpu__time_duration.sum", 0); p[2] += 1
out = {"config": cfg, "source": src, "dram_bytes": q_bytes, "serialized_time_s": q_time,
       "per_kernel": {k: {"dram_bytes": v[0], "time_s": v[1], "launches": v[2]} for k, v in per.items()},
       "note": "ncu replays kernels serialised with cold caches; the bytes are per search call"}
dst = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                   f"query_phase_traffic_config{cfg}.json")
json.dump(out, open(dst, "w"), indent=1)
print(json.dumps(out, indent=1))
