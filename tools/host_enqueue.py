#!/usr/bin/env python
"""Host time to enqueue one search (no synchronisation) vs its GPU time, config 2."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1906_12211_b200 as pfg  # noqa: E402
import synth  # noqa: E402

c = synth.CONFIGS[2]
data, q = synth.config_data(2)
dev = torch.device("cuda:0")
X, Q = torch.from_numpy(data).to(dev), torch.from_numpy(q).to(dev)
idx = pfg.Index(X, c["budget"], c["family"], seed=1)
ids = torch.empty((len(q), 10), dtype=torch.int64, device=dev)
sims = torch.empty((len(q), 10), dtype=torch.float32, device=dev)
for _ in range(10):
    idx.search(Q, 10, 0.9, out=(ids, sims))
torch.cuda.synchronize()
host, gpu = [], []
for _ in range(20):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    idx.search(Q, 10, 0.9, out=(ids, sims))
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    host.append((t1 - t0) * 1e3)
    gpu.append(e0.elapsed_time(e1))
print("host enqueue ms: median %.3f; gpu ms: median %.3f" % (sorted(host)[10], sorted(gpu)[10]))
