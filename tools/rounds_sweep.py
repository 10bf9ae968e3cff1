#!/usr/bin/env python
"""Queries/s of one config for several blind-round counts (search option `rounds`), one build."""
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
ap.add_argument("--rounds", default="3,5,7,9")
a = ap.parse_args()
c = synth.CONFIGS[a.config]
n = c.get("shard_n", c["n"])
data, q = synth.config_data(a.config, n=n)
dev = torch.device("cuda:0")
X, Q = torch.from_numpy(data).to(dev), torch.from_numpy(q).to(dev)
del data
opts = dict(strategy=c["strategy"])
if c["reps"]:
    opts["reps"] = c["reps"]
idx = pfg.Index(X, c["budget"] or 0, c["family"], seed=1, **opts)
for r in [int(x) for x in a.rounds.split(",")]:
    for _ in range(4):
        idx.search(Q, c["k"], c["recall"], rounds=r)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        idx.search(Q, c["k"], c["recall"], rounds=r)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"config {a.config} rounds {r}: {ms:.3f} ms/search, {len(q) / ms * 1e3 / 1e6:.3f} M q/s", flush=True)
