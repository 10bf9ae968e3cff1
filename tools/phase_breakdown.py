#!/usr/bin/env python
"""Per-phase times of one search (timing = 2: CUDA events between the phases' launches) after a few
warm-up searches, for a config; --rounds 200 makes every round a blind (phase-timed) round.

  python tools/phase_breakdown.py --config 4 --rounds 200
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1906_12211_b200 as pfg  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--warm", type=int, default=3)
ap.add_argument("--wide", type=int, default=0)
ap.add_argument("--rounds", type=int, default=0)
a = ap.parse_args()
c = synth.CONFIGS[a.config]
dev = torch.device("cuda:0")
data, q = synth.config_data(a.config)
X = torch.from_numpy(data).to(dev)
Q = torch.from_numpy(q).to(dev)
opts = dict(strategy=c["strategy"])
if c["reps"]:
    opts["reps"] = c["reps"]
idx = pfg.Index(X, c["budget"] or 0, c["family"], seed=1, **opts)
for _ in range(a.warm):
    idx.search(Q, c["k"], c["recall"], wide=a.wide, rounds=a.rounds)
torch.cuda.synchronize()
idx.search(Q, c["k"], c["recall"], timing=2, wide=a.wide, rounds=a.rounds)
torch.cuda.synchronize()
t = idx.last_timing()
print(json.dumps({"config": a.config, "prep_ms": t[0], "kernel_ms": t[1], "launches": t[3],
                  "phases_ms": {k: round(v, 3) for k, v in idx.last_phases().items()}}))
