#!/usr/bin/env python
"""Developer experiment: does splitting the query batch into two concurrent pipelines help?
Two indexes over the same data (same seed, so identical tables), each searching half the queries
on its own stream, against one index searching all of them.

  python tools/pipe_exp.py [--config 2] [--iters 20] [--parts 2]
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
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--parts", type=int, default=2)
a = ap.parse_args()
c = synth.CONFIGS[a.config]
dev = torch.device("cuda:0")
data, q = synth.config_data(a.config)
X = torch.from_numpy(data).to(dev)
Q = torch.from_numpy(q).to(dev)
opts = dict(strategy=c["strategy"])
if c["reps"]:
    opts["reps"] = c["reps"]
P = a.parts
idx = [pfg.Index(X, c["budget"] or 0, c["family"], seed=1, **opts) for _ in range(P)]
nq = Q.shape[0]
cuts = [nq * i // P for i in range(P + 1)]
parts = [Q[cuts[i]:cuts[i + 1]].contiguous() for i in range(P)]
streams = [torch.cuda.Stream() for _ in range(P)]


def one():
    return idx[0].search(Q, c["k"], 0.9)


def split_seq():
    return [idx[0].search(parts[i], c["k"], 0.9) for i in range(P)]


def split_conc():
    cur = torch.cuda.current_stream()
    ev = torch.cuda.Event()
    ev.record(cur)
    outs = []
    for i in range(P):
        streams[i].wait_event(ev)
        with torch.cuda.stream(streams[i]):
            outs.append(idx[i].search(parts[i], c["k"], 0.9))
    for i in range(P):
        cur.wait_stream(streams[i])
    return outs


def timeit(fn):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.iters


ids_full, _ = one()
outs = split_conc()
torch.cuda.synchronize()
same = all(torch.equal(outs[i][0], ids_full[cuts[i]:cuts[i + 1]]) for i in range(P))
print(f"config {a.config}: results of the split equal the single search: {same}")
for name, fn in (("one search", one), (f"{P} parts sequential", split_seq), (f"{P} parts concurrent", split_conc),
                 ("one search", one)):
    ms = timeit(fn)
    print(f"{name:>24}: {ms:.3f} ms/step  {nq / ms / 1e3:.3f} M q/s")
