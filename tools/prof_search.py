#!/usr/bin/env python
"""Profiling driver: build a config index, warm up, then run ONE search inside
cudaProfilerStart/Stop so `ncu --profile-from-start off` captures only the search's kernels.

  ncu --profile-from-start off --metrics gpu__time_duration.sum --csv python tools/prof_search.py --engine 0
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
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--engine", type=int, default=0)
ap.add_argument("--recall", type=float, default=0.9)
ap.add_argument("--rep-chunk", type=int, default=16)
ap.add_argument("--nq", type=int, default=0)
ap.add_argument("--warm", type=int, default=2)
ap.add_argument("--timing", type=int, default=1, help="5: the fused kernel's per-phase cycle counters (stderr)")
a = ap.parse_args()

c = synth.CONFIGS[a.config]
dev = torch.device("cuda:0")
data, q = synth.config_data(a.config, nq=a.nq or None)
X = torch.from_numpy(data).to(dev)
Q = torch.from_numpy(q).to(dev)
opts = dict(strategy=c["strategy"])
if c["reps"]:
    opts["reps"] = c["reps"]
idx = pfg.Index(X, c["budget"] or 0, c["family"], seed=1, **opts)
so = dict(rep_chunk=a.rep_chunk, engine=a.engine, timing=True)
for _ in range(a.warm):
    idx.search(Q, c["k"], a.recall, **so)
torch.cuda.synchronize()
torch.cuda.profiler.start()
idx.search(Q, c["k"], a.recall, **dict(so, timing=a.timing))
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("timing (prep_ms, kernel_ms, ?, launches):", idx.last_timing())
