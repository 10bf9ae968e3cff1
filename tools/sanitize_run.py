#!/usr/bin/env python
"""Small searches for compute-sanitizer (memcheck / racecheck / synccheck): config 1 (SimHash) and a
FHT-CP index, one engine, with wide queries and the device-side loop on for engine 0.

  compute-sanitizer --tool racecheck python tools/sanitize_run.py --engine 0
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1906_12211_b200 as pfg  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--engine", type=int, default=0)
a = ap.parse_args()
dev = torch.device("cuda:0")
d1, q1 = synth.config_data(1, n=10000, nq=100)
d2, q2 = synth.config_data(2, n=20000, nq=64)
cases = [("simhash", d1, q1, dict(reps=32)), ("fht_cp", d2, q2, dict(reps=40))]
for fam, d, q, bo in cases:
    idx = pfg.Index(torch.from_numpy(d).to(dev), 0, fam, seed=1, **bo)
    Q = torch.from_numpy(q).to(dev)
    runs = [dict()]
    if a.engine == 0:
        runs.append(dict(wide=40, loop_min=1, loop_max=1000000, rounds=2))
    for kw in runs:
        for recall in (0.9, 0.99):
            ids, sims, st = idx.search(Q, 10, recall, stats=True, engine=a.engine, rep_chunk=8, **kw)
            torch.cuda.synchronize()
    idx.close()
print("sanitize run ok, engine", a.engine)
