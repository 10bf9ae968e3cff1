#!/usr/bin/env python
"""Summarise an ncu --set full report of k_query into profiles/ (JSON): DRAM bytes, duration,
throughput, occupancy, L1/L2 hit rates and the top stall reasons."""
import csv
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, u, v = r[0], r[1], r[2]
m = {name: (v[i], u[i]) for i, name in enumerate(h)}


def f(name):
    try:
        return float(m[name][0].replace(",", ""))
    except Exception:
        return None


def scale(name, unit_mult):
    x = f(name)
    unit = m.get(name, ("", ""))[1]
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6,
            "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1}.get(unit, 1)
    return None if x is None else x * mult / unit_mult


stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): f(k) for k in h
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
tot = sum(x for x in stalls.values() if x)
top = sorted(((k, x / tot) for k, x in stalls.items() if x), key=lambda t: -t[1])[:8]
res = {
    "source": rep,
    "kernel": [n for n in h if n == "Kernel Name"] and m["Kernel Name"][0],
    "duration_s": scale("gpu__time_duration.sum", 1),
    "dram_bytes_read": scale("dram__bytes_read.sum", 1),
    "dram_bytes_write": scale("dram__bytes_write.sum", 1),
    "dram_throughput_pct_of_peak": f("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    "sm_throughput_pct": f("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    "warps_active_per_sm": f("sm__warps_active.avg.per_cycle_active"),
    "registers_per_thread": f("launch__registers_per_thread"),
    "grid": f("launch__grid_size"),
    "l1_hit_pct": f("l1tex__t_sector_hit_rate.pct"),
    "l2_hit_pct": f("lts__t_sector_hit_rate.pct"),
    "instructions": f("smsp__inst_executed.sum"),
    # FMA pipe (hashing projections: the north star asks for FMA-pipe utilisation against peak)
    "fma_pipe_active_pct": f("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
    "fma_inst_pct": f("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
    "fp32_flops_per_s": (lambda a, b: a / b if a and b else None)(
        (f("smsp__sass_thread_inst_executed_op_ffma_pred_on.sum") or 0) * 2
        + (f("smsp__sass_thread_inst_executed_op_fadd_pred_on.sum") or 0)
        + (f("smsp__sass_thread_inst_executed_op_fmul_pred_on.sum") or 0),
        scale("gpu__time_duration.sum", 1)),
    "top_stalls_share": dict(top),
}
res["dram_gbs"] = (res["dram_bytes_read"] + res["dram_bytes_write"]) / res["duration_s"] / 1e9
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
