#!/usr/bin/env python
"""Small searches through every engine / mode for compute-sanitizer (tools/sanitize.sh): SimHash
(config 1 shape) and FHT-CP (config 2 shape), engines 0/1/2, one and two round pipelines, wide
queries with the device-side loop, 16-bit rows with the re-rank.  Checks the results against each
other (the sanitizer reports the memory / race / sync errors)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1906_12211_b200 as pfg  # noqa: E402
import synth  # noqa: E402

small = len(sys.argv) > 1 and sys.argv[1] == "small"
dev = torch.device("cuda:0")
runs = 0
for cfg, fam, n, nq in ((1, "simhash", 3000 if small else 10000, 48 if small else 100),
                        (2, "fht_cp", 4000 if small else 20000, 40 if small else 100)):
    data, q = synth.config_data(cfg, n=n, nq=nq)
    for storage in ("f32", "i16"):
        g = pfg.Index(torch.from_numpy(data).to(dev), 0, fam, seed=1, reps=24, storage=storage)
        Q = torch.from_numpy(q).to(dev)
        ref = None
        for kw in (dict(engine=0), dict(engine=1), dict(engine=2), dict(engine=0, pipelines=2),
                   dict(engine=0, pipelines=2, rounds=1), dict(engine=0, wide=2, loop_min=1, loop_max=1 << 20),
                   dict(engine=0, rounds=1, wide=-1)):
            ids, sims = g.search(Q, 10, 0.9, rep_chunk=8, **kw)
            torch.cuda.synchronize()
            runs += 1
            if ref is None:
                ref = ids.cpu().numpy()
            else:
                assert np.array_equal(ids.cpu().numpy(), ref), (cfg, storage, kw)
print(f"sanitize_run: {runs} searches, results identical across engines and modes")
