#!/usr/bin/env python
"""Benchmark of the batched LSH-forest k-NN query path (BASELINE.json metric: queries/s at >= 0.9
recall, k = 10, 1M x 100-d angular; achieved HBM GB/s).

A "step" is one pass of the hot path over one batch: pfg_search over all nq queries of the
workload (normalise, hash, sketch, adaptive query kernel with its stop rule; plus the NCCL
all-gather and merge kernel when N > 1).  The index is built once before timing (its time is
reported as build_s).  Inputs are resident in HBM when a timed step starts; L2 is flushed (512 MiB
write) between timed steps.  `e2e` repeats the measurement through the same C-ABI call with
pinned HOST query/result buffers (host<->device copies inside the timed region).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--recall 0.9]
  python bench.py --impl reference ...   # the CPU oracle (test infrastructure) on the host cores
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "queries/s at >=0.9 recall, k=10, 1Mx100-d angular; achieved HBM GB/s"
WORKLOAD_NOTE = {2: " (Gaussian-mixture stand-in for GloVe-1M)",
                 3: " (planted-partner stand-in for the paper's SYNTHETIC set)",
                 6: " (the paper's SYNTHETIC construction, PAPER.md:424-439)"}


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "_fallback": True}


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled every 200 ms during the timed region"""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.rows, self.proc = gpu, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "200", "-i", str(self.gpu)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        sm = []
        mx = None
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
            except ValueError:
                continue
            for nm, v in zip(names, r[3:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------- helpers
def cfg_desc(cfg: int):
    c = synth.CONFIGS[cfg]
    return c


def ground_truth(data_t, q_t, k):
    """exact top-k by fp32 inner products of the normalised rows (torch, TF32 off; measurement
    tool, not part of the path), in blocks of queries x rows.  Returns (ids [nq,k], kth sims [nq])."""
    import torch
    torch.backends.cuda.matmul.allow_tf32 = False
    x = data_t / data_t.norm(dim=1, keepdim=True)
    q = q_t / q_t.norm(dim=1, keepdim=True)
    qb, xb = 1024, 1 << 21
    ids, kth = [], []
    for s in range(0, q.shape[0], qb):
        bv = bi = None
        for r0 in range(0, x.shape[0], xb):
            S = q[s:s + qb] @ x[r0:r0 + xb].T
            v, i = torch.topk(S, min(k, S.shape[1]), dim=1)
            i = i + r0
            if bv is not None:
                v = torch.cat([bv, v], 1)
                i = torch.cat([bi, i], 1)
                v, o = torch.topk(v, k, dim=1)
                i = torch.gather(i, 1, o)
            bv, bi = v, i
            del S
        ids.append(bi)
        kth.append(bv[:, -1])
    return torch.cat(ids), torch.cat(kth), x, q


def recall_of(ids_t, truth_kth, xn, qn, k):
    """tie-tolerant recall@k: a returned id counts if its exact sim >= true k-th sim - 1e-5"""
    import torch
    ids = ids_t.clamp(min=0)
    s = torch.einsum("qd,qkd->qk", qn, xn[ids])
    hit = (s >= truth_kth[:, None] - 1e-5) & (ids_t >= 0)
    return float(hit.float().sum() / (k * ids_t.shape[0]))


def alg_bytes(stats, d, M, k, row_bytes=None):
    """algorithmic bytes of the query kernel: per query
    B_q = 16 E + r S + 8 P + r + 8M + 12k  (E retrieved 16-byte table entries, S evaluated rows of
    r = 4d bytes (fp32; 2d for the int16 storage of R-25), P binary-search probes; plus the query
    row, its sketches and the outputs)"""
    r = 4 * d if row_bytes is None else row_bytes
    em = stats["emitted"].astype(np.float64)
    ev = stats["evaluated"].astype(np.float64)
    pr = stats["probes"].astype(np.float64)
    b = 16 * em + r * ev + 8 * pr + r + 8 * M + 12 * k
    return float(b.sum())


def profiled_traffic(cfg):
    """DRAM bytes (read + write) of the query phase of one search call, summed over its kernels,
    from the committed ncu capture (tools/ncu_traffic.py), if present for this config"""
    path = os.path.join(ROOT, "profiles", f"query_phase_traffic_config{cfg}.json")
    try:
        j = json.load(open(path))
        return float(j["dram_bytes"]), os.path.relpath(path, ROOT)
    except Exception:
        return None, None


# ---------------------------------------------------------------------------- reference arm
def profiled_ksims_traffic(cfg):
    """DRAM bytes per k_sims launch (all launches of one search, ncu --set full) if captured"""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", f"ksims_traffic_config{cfg}.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        return json.load(f)


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_index(cfg):
    """the CPU oracle (test infrastructure) over a config's data, repetition tables built lazily;
    L comes from the config record (the product's cost model is not loaded, R-11)"""
    import oracle as O
    c = synth.CONFIGS[cfg]
    data, q = synth.config_data(cfg, n=c.get("shard_n"))
    fam = {"simhash": O.HP, "fht_cp": O.FHTCP, "cp": O.CP}[c["family"]]
    strat = O.POOL if c["strategy"] == "pool" else O.INDEPENDENT
    return O.OracleIndex(data, fam, L=c["reps"] or c["L"], seed=1, strategy=strat, lazy=True), q


def oracle_recall(X, qs, ids, k):
    import oracle as O
    bi, _ = O.bruteforce(X.data(), O.normalize(qs), k)
    return float(np.mean([len(set(a) & set(b)) / k for a, b in zip(ids.tolist(), bi.tolist())]))


def config_record(args, c, n, nq, reps, world=1, sharded=False, replicas=False):
    """the `config` object of the JSON line: the workload and the search options, the same for the
    product arm and the reference arm (which runs the oracle on this workload with these options;
    engine / rounds / pipelines / l2 describe the product's launch and are carried verbatim)"""
    weak = "shard_n" in c
    return {"workload": f"config{args.config}: {c['name']}" + WORKLOAD_NOTE.get(args.config, "")
            + (" [int16 fixed-point rows, R-25]" if args.storage == "i16" else "")
            + (f" ({c['shard_n']} rows per GPU)" if weak else ""),
            "n": n, "d": c["d"], "nq": nq, "k": c["k"], "recall_target": args.recall, "family": c["family"],
            "strategy": c["strategy"], "budget_bytes_per_gpu": c["budget"], "reps": reps,
            "rep_chunk": args.rep_chunk, "uniform_chunks": args.uniform_chunks, "storage": args.storage,
            "tau_rule": ["quantile (R-26)", "expected distance (R-15)"][args.tau_rule],
            "engine": args.engine, "rounds": args.rounds or 5,
            "pipelines": args.pipelines or 1,
            "l2": "flushed (512 MiB write) between timed steps",
            "parallelism": (f"data-sharded x{world}" if sharded else
                            f"query replicas x{world} (every GPU builds the whole index and answers a batch "
                            f"of {nq} queries independently; no collective on the data path)" if replicas
                            else "single GPU")}


def run_reference(args):
    """The CPU oracle as it stands (test infrastructure), timed on all host cores (OpenMP over the
    queries), each step a bounded sample of the workload's queries."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    c = synth.CONFIGS[args.config]
    nq = c["nq"]
    cores = os.cpu_count() or 1
    t0 = time.time()
    X, q = oracle_index(args.config)
    sample = args.ref_sample
    qs = q[:sample]
    X.search(qs, c["k"], args.recall, rep_chunk=args.rep_chunk, tau_rule=args.tau_rule,
             uniform_chunks=args.uniform_chunks)   # builds the repetitions it touches
    setup = time.time() - t0
    times = []
    for s in range(args.warmup + args.steps):
        t = time.perf_counter()
        ids, sims, tr = X.search(qs, c["k"], args.recall, rep_chunk=args.rep_chunk, threads=cores, tau_rule=args.tau_rule,
                                  uniform_chunks=args.uniform_chunks)
        el = time.perf_counter() - t
        if s >= args.warmup:
            times.append(el)
    tot = sum(times)
    value = args.steps * sample / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True,
        "scaling": "weak" if ("shard_n" in c or args.parallel == "queries") else "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_record(args, c, c.get("shard_n", c["n"]), nq, c["reps"] or c["L"]),
        "recall": oracle_recall(X, qs, ids, c["k"]),
        "cpu_baseline": {"value": value, "unit": "queries/s", "cores": cores, "kind": "oracle",
                         "cpu_model": cpu_model(),
                         "sample": f"first {sample} of {nq} queries per step, OpenMP over the queries on {cores} "
                                   f"host threads, lazily built oracle index ({setup:.0f} s setup untimed)"},
        "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline_leg(cfg, recall, rep_chunk, sample1, sample_all):
    """the oracle on the host cores: (i) one thread on the first `sample1` queries (the paper's
    protocol), (ii) OpenMP over all cores on the first `sample_all` queries"""
    c = synth.CONFIGS[cfg]
    cores = os.cpu_count() or 1
    if c.get("shard_n", c["n"]) * c["d"] > 400_000_000:
        # the oracle's index setup alone (2048 sketch projections per point) exceeds the bounded
        # budget of this leg; the reference arm (--impl reference) times it separately
        return {"value": None, "unit": "queries/s", "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
                "sample": f"not run: config {cfg}'s oracle setup ({c['n']} x {c['d']}) exceeds the bounded CPU budget"}
    t0 = time.time()
    X, q = oracle_index(cfg)
    qa = q[:sample_all]
    X.search(qa, c["k"], recall, rep_chunk=rep_chunk)    # builds the repetitions the sample touches
    setup = time.time() - t0
    t = time.perf_counter()
    X.search(q[:sample1], c["k"], recall, rep_chunk=rep_chunk, threads=1)
    one = sample1 / (time.perf_counter() - t)
    t = time.perf_counter()
    ids, _, _ = X.search(qa, c["k"], recall, rep_chunk=rep_chunk, threads=cores)
    allc = sample_all / (time.perf_counter() - t)
    return {"value": allc, "unit": "queries/s", "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
            "sample": f"first {sample_all} of {c['nq']} queries, OpenMP over the queries on {cores} host threads; "
                      f"lazily built oracle index, {setup:.0f} s setup untimed",
            "recall": oracle_recall(X, qa, ids, c["k"]),
            "single_thread": {"value": one, "unit": "queries/s", "cores": 1,
                              "sample": f"first {sample1} queries, one thread (the paper's protocol, PAPER.md:362-363)"}}


# ---------------------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--recall", type=float, default=0.9)
    ap.add_argument("--rep-chunk", type=int, default=16)
    ap.add_argument("--nq", type=int, default=0, help="override the query count")
    ap.add_argument("--ref-sample", type=int, default=500, help="queries per step of the reference arm")
    ap.add_argument("--cpu-sample", type=int, default=1000, help="queries of the single-thread CPU leg (BASELINE.md: the first 1 000)")
    ap.add_argument("--cpu-sample-all", type=int, default=2000, help="queries of the all-cores CPU leg")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--engine", type=int, default=0, help="0 = phase-split rounds + fused kernel, 1 = fused kernel only, 2 = chunk rounds + fused kernel")
    ap.add_argument("--uniform-chunks", action="store_true", help="first chunk R repetitions long (R-17 option)")
    ap.add_argument("--rounds", type=int, default=0, help="bulk rounds before the fused kernel (0 = library default)")
    ap.add_argument("--pipelines", type=int, default=0, help="engine 0 round pipelines: 0 = library default (one), 1, 2")
    ap.add_argument("--tau-rule", type=int, default=0, help="0 = quantile filter threshold (R-26), 1 = expected distance (R-15)")
    ap.add_argument("--parallel", default="data", choices=["data", "queries"],
                    help="N > 1: data-sharded (the default, SURVEY 8(e): each GPU indexes n/N rows -- 12.5M rows per GPU "
                         "for config 5 -- every query on every GPU, distributed query hashing, NCCL all-gather + merge), "
                         "or query replicas (each GPU the whole index and a query batch of its own; query-parallel "
                         "throughput, no collective)")
    ap.add_argument("--no-distributed-prep", action="store_true",
                    help="data-sharded mode: every rank hashes every query (instead of 1/N and an all-gather)")
    ap.add_argument("--storage", default="f32", choices=["f32", "i16"],
                    help="rows for the inner products: fp32, or the paper's 16-bit fixed point (R-25)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import paper_1906_12211_b200 as pfg
    from paper_1906_12211_b200.sharded import ReplicatedIndex, ShardedIndex, shard_range

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    c = synth.CONFIGS[args.config]
    d, k = c["d"], c["k"]
    # config 5 is weak-scaled (BASELINE: 12.5M rows per GPU); the others split their n rows
    weak = "shard_n" in c
    mode = args.parallel
    sharded = world > 1 and mode == "data"
    replicas = world > 1 and mode == "queries"
    n = c["shard_n"] * world if (weak and sharded) else c["n"] if not weak else c["shard_n"]
    nq = args.nq or c["nq"]
    lo, hi = shard_range(n, world, rank) if sharded else (0, n)
    data_np, q_np = synth.config_data(args.config, n=hi - lo, nq=nq, row0=lo)
    data = torch.from_numpy(data_np).to(dev)
    q = torch.from_numpy(q_np).to(dev)
    del data_np

    opts = dict(strategy=c["strategy"], storage=args.storage)
    if c["reps"]:
        opts["reps"] = c["reps"]
    torch.cuda.synchronize()
    t0 = time.time()
    idx = (ShardedIndex(data, lo, c["budget"] or 0, c["family"], seed=1, **opts) if sharded or world == 1
           else ReplicatedIndex(data, c["budget"] or 0, c["family"], seed=1, **opts))
    torch.cuda.synchronize()
    build_s = time.time() - t0
    info = idx.index.info

    # ground truth (global): shard-local exact top-k, gathered and merged like the search
    t_ids, t_kth, xn, qn = ground_truth(data, q, k)
    if sharded:
        from paper_1906_12211_b200.sharded import gather_merge
        sims_local = torch.einsum("qd,qkd->qk", qn, xn[t_ids])
        _, ms = gather_merge(t_ids + lo, sims_local.contiguous())
        t_kth = ms[:, -1].contiguous()

    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    sopts = dict(rep_chunk=args.rep_chunk, timing=True, engine=args.engine, uniform_chunks=args.uniform_chunks,
                 rounds=args.rounds, tau_rule=args.tau_rule, pipelines=args.pipelines)
    if sharded and not args.no_distributed_prep:
        sopts["distributed_prep"] = True

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
    t_w = time.time()
    while True:  # warm-up: at least `warmup` steps and ~1 s so the clock sampler is running
        for _ in range(args.warmup):
            idx.search(q, k, args.recall, **sopts)
        torch.cuda.synchronize()
        if time.time() - t_w > 1.0:
            break
    step_ms, kern_ms, prep_ms = [], [], []
    phase_ms = {}
    launches = 0
    stats = None
    # timing = 3: CUDA events around every bulk k_sims launch of the timed steps (the dominant
    # kernel's roofline below), accumulated by the library on the search stream
    sopts_t = dict(sopts, timing=3)
    idx.index.kernel_timing(reset=True)
    # the K steps are enqueued back to back (barrier + synchronize before and after them only): each
    # step's search is bracketed by CUDA events on the stream, the L2 flush between steps is outside
    # them, and the host enqueues the next step while the GPU runs the current one
    barrier()
    evs = []
    for s in range(args.steps):
        flush.fill_(s & 0xff)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        res = idx.search(q, k, args.recall, **sopts_t)
        e1.record(stream)
        evs.append((e0, e1))
    barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    nl = idx.index.last_timing()[3]
    launches = (nl + (1 if sharded else 0)) * args.steps
    clocks = sampler.stop() if sampler else None
    # preparation / query-phase split of a search (untimed searches with events between them)
    for _ in range(3):
        idx.search(q, k, args.recall, **sopts)
        pm, km, _, _ = idx.index.last_timing()
        prep_ms.append(pm)
        kern_ms.append(km)
    ksims_ms, ksims_launches = idx.index.kernel_timing(reset=True)
    # per-query counters (algorithmic bytes, stop depths) from one more, untimed search of the same
    # batch; the search is deterministic, so they are the counters of the timed steps
    ids, sims, stats = idx.search(q, k, args.recall, stats=True, **sopts)[:3]
    rstats = idx.index.round_stats() if args.engine in (0, 2) else None
    # per-phase breakdown of the query kernels from untimed searches with events between phases
    for _ in range(3):
        idx.search(q, k, args.recall, **dict(sopts, timing=2))
        for key, v in idx.index.last_phases().items():
            phase_ms[key] = phase_ms.get(key, 0.0) + v / 3
    tot_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([tot_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
    rec = recall_of(ids, t_kth, xn, qn, k) if not sharded else None
    if sharded:
        # recall against the merged global truth: check returned ids' exact sims on their owning rank
        owned = (ids >= lo) & (ids < hi)
        loc = (ids - lo).clamp(0, hi - lo - 1)
        s_exact = torch.einsum("qd,qkd->qk", qn, xn[loc]) * owned
        dist.all_reduce(s_exact)
        hit = (s_exact >= t_kth[:, None] - 1e-5) & (ids >= 0)
        rec = float(hit.float().sum() / (k * nq))

    # e2e: same call with pinned host buffers (H2D of queries, D2H of ids + sims inside the region)
    e2e = None
    if not args.no_e2e:
        qh = q.cpu().pin_memory()
        ih = torch.empty((nq, k), dtype=torch.int64).pin_memory()
        sh = torch.empty((nq, k), dtype=torch.float32).pin_memory()
        e2e_ms = []
        for s in range(args.warmup + args.steps):
            flush.fill_(s & 0xff)
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            idx.index.search(qh.numpy(), k, args.recall, out=(ih.numpy(), sh.numpy()), stream=stream,
                             **{o: v for o, v in sopts.items() if o != "distributed_prep"})
            e1.record(stream)
            barrier()
            if s >= args.warmup:
                e2e_ms.append(e0.elapsed_time(e1))
        et = sum(e2e_ms)
        if world > 1:
            t = torch.tensor([et], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            et = float(t.item())
        e2e = {"value": args.steps * nq * (world if replicas else 1) / (et / 1e3), "unit": "queries/s",
               "h2d_bytes_per_step": nq * d * 4 * (world if replicas else 1),
               "d2h_bytes_per_step": nq * k * 12 * (world if replicas else 1)}

    if rank == 0:
        pk = peaks()
        ab = alg_bytes(stats, d, info["sketch_words"], k, row_bytes=2 * d if args.storage == "i16" else 4 * d)
        kern_s = statistics.mean(kern_ms) / 1e3
        achieved = ab / kern_s / 1e9
        traffic, traffic_src = profiled_traffic(args.config) if args.storage == "f32" else (None, None)
        # the dominant kernel (k_sims, the bulk similarity gathers): algorithmic bytes per launch =
        # the rows its timed launches computed (the blind rounds' launches, which timing = 3 brackets
        # with CUDA events; rows computed inside the device-side loop are not counted) x the 4d bytes
        # of a row (4d per evaluated row; the 16 B of pool entry per row are overhead),
        # over the average duration of those launches
        ksims_roofline = None
        if rstats and ksims_launches:
            row_b = 2 * d if args.storage == "i16" else 4 * d
            per_launch = rstats["sims_rows_blind"] * args.steps * row_b / ksims_launches
            launch_s = ksims_ms / ksims_launches / 1e3
            frac = per_launch / launch_s / 1e9 / pk["hbm_gbs"]
            ks_tr = profiled_ksims_traffic(args.config) if args.storage == "f32" else None
            ksims_roofline = {"bound": "hbm", "kernel": "k_sims (bulk candidate-row gathers + dot products, "
                                                        "the largest share of the query phase)",
                              "achieved": per_launch / launch_s / 1e9, "peak": pk["hbm_gbs"], "unit": "GB/s",
                              "frac": frac,
                              "traffic": ks_tr["dram_bytes_per_launch"] if ks_tr else None,
                              "traffic_source": ks_tr["source"] if ks_tr else None,
                              "alg_bytes_per_launch": per_launch, "alg_bytes_unit": f"{row_b} B per evaluated row",
                              "launch_ms": launch_s * 1e3, "launches": ksims_launches,
                              "share_of_query_phase": ksims_ms / args.steps / statistics.mean(kern_ms),
                              "peak_source": "MEASURED_PEAKS.json hbm_gbs" if not pk.get("_fallback") else "fallback"}
            if frac > 1.0:
                # more algorithmic bytes than the DRAM can deliver: the accounting is wrong (or rows
                # came from L2); flagged, never reported as a fraction of the roofline
                print(f"bench: k_sims roofline fraction {frac:.3f} exceeds 1 (accounting error)", file=sys.stderr)
                ksims_roofline["frac_invalid"] = True
        cpu = None
        if not args.no_cpu_baseline:
            try:
                cpu = cpu_baseline_leg(args.config, args.recall, args.rep_chunk, args.cpu_sample, args.cpu_sample_all)
            except Exception as e:  # pragma: no cover
                cpu = {"value": None, "unit": "queries/s", "cores": 1, "kind": "oracle", "sample": f"failed: {e}"}
        line = {
            "metric": METRIC,
            "value": args.steps * nq * (world if replicas else 1) / (tot_ms / 1e3),
            "unit": "queries/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": tot_ms / args.steps,
            "higher_is_better": True,
            "scaling": "weak" if (weak or mode == "queries") else "strong",
            "vs_baseline": None,
            "dtype": "f32" if args.storage == "f32" else "i16 rows (int32 dot), f32 hashing",
            "data": "synthetic",
            "config": config_record(args, c, n, nq, info["reps"], world, sharded, replicas),
            "recall": rec,
            "build_s": build_s,
            "roofline": ksims_roofline,
            # the whole step (preparation included): all algorithmic bytes of the search over ms_per_step
            "roofline_step": {"bound": "hbm", "achieved": ab / (tot_ms / args.steps / 1e3) / 1e9, "peak": pk["hbm_gbs"],
                              "unit": "GB/s", "frac": ab / (tot_ms / args.steps / 1e3) / 1e9 / pk["hbm_gbs"],
                              "alg_bytes_per_step": ab},
            "roofline_query_phase": {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                         "frac": achieved / pk["hbm_gbs"], "traffic": traffic, "traffic_source": traffic_src,
                         "kernel": "query phase: bulk rounds (k_expand, k_scan, k_dedupe, k_sims, k_merge) "
                                   "+ fused tail (k_query), one search call",
                         "kernel_ms": statistics.mean(kern_ms), "phases_ms_untimed": phase_ms,
                         "prep_ms": statistics.mean(prep_ms), "alg_bytes_per_query": ab / nq,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs" if not pk.get("_fallback") else "fallback"},
            "round_stats": rstats,
            "counters": {"emitted_per_q": float(np.mean(stats["emitted"])),
                         "evaluated_per_q": float(np.mean(stats["evaluated"])),
                         "filtered_per_q": float(np.mean(stats["filtered"])),
                         "dups_per_q": float(np.mean(stats["dups"])),
                         "i_stop_mean": float(np.mean(stats["i_stop"])),
                         "j_stop_mean": float(np.mean(stats["j_stop"])),
                         "j_stop_p50_p90_p99_max": [float(np.percentile(stats["j_stop"], q)) for q in (50, 90, 99, 100)],
                         "evaluated_p99_max": [float(np.percentile(stats["evaluated"], 99)),
                                               float(np.max(stats["evaluated"]))],
                         "bitmap_mode_queries": int(np.sum((stats["flags"] & 8) != 0))},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
