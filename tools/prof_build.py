#!/usr/bin/env python
"""Profiling driver for the index build: one config build inside cudaProfilerStart/Stop, so that
`ncu --profile-from-start off` sees only the build's kernels (k_normalize, the sketch GEMM, the
repetition hashing k_fht_keys / k_hp_bits_tc, the CUB sorts, k_entries, k_prefix).

  ncu --profile-from-start off --kernel-name regex:k_fht_keys --set full python tools/prof_build.py
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1906_12211_b200 as pfg  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
a = ap.parse_args()
c = synth.CONFIGS[a.config]
data, _ = synth.config_data(a.config, nq=1)
X = torch.from_numpy(data).to(torch.device("cuda:0"))
opts = dict(strategy=c["strategy"])
if c["reps"]:
    opts["reps"] = c["reps"]
pfg.Index(X, c["budget"] or 0, c["family"], seed=2, **opts).close()   # warm-up (module load, allocator)
torch.cuda.synchronize()
torch.cuda.profiler.start()
t = time.perf_counter()
idx = pfg.Index(X, c["budget"] or 0, c["family"], seed=1, **opts)
torch.cuda.synchronize()
print(f"build: {time.perf_counter() - t:.3f} s, L = {idx.info['reps']}")
torch.cuda.profiler.stop()
