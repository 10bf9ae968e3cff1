#!/usr/bin/env python
"""How much row reuse does a locality order expose?  Evaluated-id traces of config 2's batch: the
number of distinct rows in consecutive blocks of B queries (an ideal cache holding one block's
rows) relative to all evaluations, for the given order and for queries sorted by their
repetition-0 code."""
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
ids, sims, st, tr = idx.search(torch.from_numpy(q).to(dev), 10, 0.9, stats=True, trace_cap=2048)
ev = st["evaluated"].astype(np.int64)
tot = int(ev.sum())
rows = [tr[r, :min(2048, ev[r])] for r in range(len(q))]
for name, o in (("given", np.arange(len(q))), ("rep0_code", np.argsort(codes[:, 0], kind="stable")),
                ("code_012", np.lexsort((codes[:, 2], codes[:, 1], codes[:, 0])))):
    out = []
    for B in (8, 64, 460, 2000):
        u = 0
        for s in range(0, len(q), B):
            u += len(np.unique(np.concatenate([rows[r] for r in o[s:s + B]])))
        out.append(f"B={B}: {u / tot:.3f}")
    print(name, "distinct/evaluated", ", ".join(out), flush=True)
