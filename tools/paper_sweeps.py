#!/usr/bin/env python
"""Counter reproductions of the paper's parameter studies on the config-2 stand-in:
recall targets (BASELINE config 2: .5/.9/.99), the filter's eps and the filter off (Fig. 2,
PAPER.md:504-532), the memory budget (Fig. 3) and the segment size B (Table 3,
PAPER.md:920-934).  For each setting: queries/s (CUDA events around the search, inputs resident,
median of 5), measured recall@k against the exact top-k, and the per-query counters.

  python tools/paper_sweeps.py [--out profiles/r02/sweeps_config2.jsonl]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1906_12211_b200 as pfg  # noqa: E402
import synth  # noqa: E402
from bench import ground_truth, recall_of  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02", "sweeps_config2.jsonl"))
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()

c = synth.CONFIGS[2]
dev = torch.device("cuda:0")
data, q = synth.config_data(2)
X = torch.from_numpy(data).to(dev)
Q = torch.from_numpy(q).to(dev)
k = c["k"]
_, kth, xn, qn = ground_truth(X, Q, k)
lines = []


def run(idx, label, recall, **sopts):
    ts = []
    for r in range(a.reps + 1):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        ids, sims = idx.search(Q, k, recall, **sopts)[:2]
        e1.record()
        torch.cuda.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1))
    ids, sims, st = idx.search(Q, k, recall, stats=True, **sopts)
    ms = statistics.median(ts)
    line = {"sweep": label, "recall_target": recall, "opts": sopts, "reps_L": idx.info["reps"],
            "queries_per_s": len(q) / (ms / 1e3), "ms": ms, "recall": recall_of(ids, kth, xn, qn, k),
            "emitted": float(np.mean(st["emitted"])), "filtered": float(np.mean(st["filtered"])),
            "dups": float(np.mean(st["dups"])), "evaluated": float(np.mean(st["evaluated"])),
            "j_stop_mean": float(np.mean(st["j_stop"])), "i_stop_mean": float(np.mean(st["i_stop"]))}
    print(json.dumps(line), flush=True)
    lines.append(line)


idx = pfg.Index(X, c["budget"], c["family"], seed=1)
for rec in (0.5, 0.9, 0.99):
    run(idx, "recall", rec)                           # the default quantile filter (R-26)
for rec in (0.5, 0.9, 0.99):
    run(idx, "recall_expected_distance", rec, tau_rule=1)
for eps in (-0.2, 0.0, 0.2, 0.5):
    run(idx, "eps", 0.9, eps=eps, tau_rule=1)         # the paper's (1 + eps) x expected distance (R-15)
run(idx, "filter_off", 0.9, use_filter=False)
for B in (1, 4, 12, 24):
    run(idx, "segment", 0.9, segment=B)
del idx
torch.cuda.empty_cache()
for gib in (1, 2, 4, 8):
    idx = pfg.Index(X, gib << 30, c["family"], seed=1)
    for rec in (0.5, 0.9):
        run(idx, f"budget_{gib}GiB", rec)
    del idx
    torch.cuda.empty_cache()
os.makedirs(os.path.dirname(a.out), exist_ok=True)
with open(a.out, "w") as f:
    for line in lines:
        f.write(json.dumps(line) + "\n")
