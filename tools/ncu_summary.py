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


def f(k):
    try:
        return float(d[k].replace(",", ""))
    except (KeyError, ValueError):
        return None


stalls = {}
for k in h:
    if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
        name = k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]
        val = f(k)
        if val and val > 0.01:
            stalls[name] = round(val, 3)
out = {
    "kernel": d.get("Kernel Name"),
    "duration_ms": (f("gpu__time_duration.sum") or 0) / 1e6,
    "sm_mhz": (f("smsp__cycles_elapsed.avg.per_second") or 0) / 1e6,
    "fp64_pipe_active_pct": f("TPC.TriageCompute.sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"),
    "alu_pipe_pct": f("TPC.TriageCompute.sm__inst_executed_pipe_alu_realtime.avg.pct_of_peak_sustained_elapsed"),
    "issue_slots_busy_pct": f("sm__inst_issued.avg.pct_of_peak_sustained_active"),
    "ipc": f("sm__inst_executed.avg.per_cycle_active"),
    "inst_executed": f("smsp__inst_executed.sum"),
    "registers": f("launch__registers_per_thread"),
    "dram_bytes_read": f("dram__bytes_read.sum"),
    "dram_bytes_write": f("dram__bytes_write.sum"),
    "stalls_cycles_per_issue": dict(sorted(stalls.items(), key=lambda x: -x[1])),
}
out["dram_bytes_per_launch"] = (out["dram_bytes_read"] or 0) + (out["dram_bytes_write"] or 0)
print(json.dumps(out, indent=1))
