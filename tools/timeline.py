#!/usr/bin/env python
"""Developer timeline of one config search (search option timing = 4): completion time of each
launch group on its stream relative to the call's first event, printed by the library to stderr.

  python tools/timeline.py [--config 2] [--engine 0]
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
ap.add_argument("--storage", default="f32", choices=["f32", "i16"])
ap.add_argument("--pipelines", type=int, default=0)
a = ap.parse_args()
c = synth.CONFIGS[a.config]
dev = torch.device("cuda:0")
data, q = synth.config_data(a.config)
X = torch.from_numpy(data).to(dev)
Q = torch.from_numpy(q).to(dev)
opts = dict(strategy=c["strategy"], storage=a.storage)
if c["reps"]:
    opts["reps"] = c["reps"]
idx = pfg.Index(X, c["budget"] or 0, c["family"], seed=1, **opts)
for _ in range(3):
    idx.search(Q, c["k"], a.recall, engine=a.engine, pipelines=a.pipelines, rep_chunk=16)
torch.cuda.synchronize()
print(f"== config {a.config} engine {a.engine}", file=sys.stderr, flush=True)
idx.search(Q, c["k"], a.recall, engine=a.engine, pipelines=a.pipelines, rep_chunk=16, timing=4)
torch.cuda.synchronize()
