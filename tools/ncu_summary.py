#!/usr/bin/env python3
"""Summarise an ncu report (k_join): pipe use, issue, stalls, DRAM bytes."""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
d = dict(zip(h, v))
units = dict(zip(h, u))
_SCALE = {  # ncu unit strings -> SI base (seconds, bytes, per second)
    "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
    "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0,
    "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
    "cycle/nsecond": 1e9, "cycle/usecond": 1e6, "cycle/msecond": 1e3, "cycle/second": 1.0,
    "hz": 1.0, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9,
}


def f(k):
    try:
        return float(d[k].replace(",", ""))
    except (KeyError, ValueError):
        return None


def si(k):
    """Value of metric k in SI base units (s, bytes, 1/s) using ncu's unit row."""
    x = f(k)
    if x is None:
        return None
    return x * _SCALE.get(units.get(k, "").strip(), 1.0)


stalls = {}
for k in h:
    if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
        name = k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]
        val = f(k)
        if val and val > 0.01:
            stalls[name] = round(val, 3)
out = {
    "kernel": d.get("Kernel Name"),
    "duration_ms": (si("gpu__time_duration.sum") or 0) * 1e3,
    "sm_mhz": (si("smsp__cycles_elapsed.avg.per_second") or 0) / 1e6,
    "fp64_pipe_active_pct": f("TPC.TriageCompute.sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"),
    "alu_pipe_pct": f("TPC.TriageCompute.sm__inst_executed_pipe_alu_realtime.avg.pct_of_peak_sustained_elapsed"),
    "issue_slots_busy_pct": f("sm__inst_issued.avg.pct_of_peak_sustained_active"),
    "ipc": f("sm__inst_executed.avg.per_cycle_active"),
    "inst_executed": f("smsp__inst_executed.sum"),
    "registers": f("launch__registers_per_thread"),
    "dram_bytes_read": si("dram__bytes_read.sum"),
    "dram_bytes_write": si("dram__bytes_write.sum"),
    "stalls_cycles_per_issue": dict(sorted(stalls.items(), key=lambda x: -x[1])),
}
out["dram_bytes_per_launch"] = (out["dram_bytes_read"] or 0) + (out["dram_bytes_write"] or 0)
print(json.dumps(out, indent=1))
