#!/usr/bin/env python
"""Experiment: does processing the batch in a locality order (queries sorted by their repetition-0
code) change the search time?  Config 2, CUDA events, L2 flushed between searches."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1906_12211_b200 as pfg  # noqa: E402
import synth  # noqa: E402

c = synth.CONFIGS[2]
dev = torch.device("cuda:0")
data, q = synth.config_data(2)
idx = pfg.Index(torch.from_numpy(data).to(dev), c["budget"], c["family"], seed=1)
codes, _ = idx.hash_queries(q)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
orders = {"given": np.arange(len(q)), "rep0_code": np.argsort(codes[:, 0], kind="stable"),
          "code_01": np.lexsort((codes[:, 1], codes[:, 0])), "random": np.random.default_rng(0).permutation(len(q))}
for name, o in orders.items():
    Q = torch.from_numpy(np.ascontiguousarray(q[o])).to(dev)
    for _ in range(5):
        idx.search(Q, 10, 0.9)
    ts = []
    for _ in range(30):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        idx.search(Q, 10, 0.9)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ids, _ = idx.search(Q, 10, 0.9)
    ph = idx.search(Q, 10, 0.9, timing=2) and idx.last_phases()
    print(f"{name}: {np.median(ts):.3f} ms (min {np.min(ts):.3f}); phases {({k: round(v, 3) for k, v in ph.items()})}", flush=True)
