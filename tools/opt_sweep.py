#!/usr/bin/env python
"""Developer sweep: one config index, then the median device time of a search of the whole query
batch under each option set given on the command line (JSON dicts of Index.search keywords), with
the stop-depth histogram of the default search.

  python tools/opt_sweep.py '{}' '{"rounds": 4}' '{"engine": 2}'
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1906_12211_b200 as pfg  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--reps", type=int, default=15)
ap.add_argument("--storage", default="f32")
ap.add_argument("sets", nargs="*")
a = ap.parse_args()
c = synth.CONFIGS[a.config]
dev = torch.device("cuda:0")
data, q = synth.config_data(a.config)
X = torch.from_numpy(data).to(dev)
Q = torch.from_numpy(q).to(dev)
opts = dict(strategy=c["strategy"])
if c["reps"]:
    opts["reps"] = c["reps"]
if a.storage == "i16":
    opts["storage"] = "i16"
idx = pfg.Index(X, c["budget"] or 0, c["family"], seed=1, **opts)
ids0, _, st = idx.search(Q, c["k"], c["recall"], stats=True)
js = st["j_stop"]
print("j_stop > 1/17/33/49/65:", [int((js > t).sum()) for t in (1, 17, 33, 49, 65)], "max", int(js.max()))
for s in a.sets or ["{}"]:
    kw = json.loads(s)
    ts = []
    for it in range(a.reps + 3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        ids, sims = idx.search(Q, c["k"], c["recall"], **kw)
        e1.record()
        torch.cuda.synchronize()
        if it >= 3:
            ts.append(e0.elapsed_time(e1))
    same = bool(torch.equal(ids.cpu(), ids0.cpu()))
    print(f"{s}: median {np.median(ts):.3f} ms  min {np.min(ts):.3f}  same_ids {same}", flush=True)
