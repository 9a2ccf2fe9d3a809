"""Summarise ncu --set full reports (raw page) into profiles/ncu_summary.json.

    python tools/ncu_summary.py C2=gpurun_out/prof_c2_r01.ncu-rep C3=gpurun_out/prof_c3_r01.ncu-rep
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = {
    "time_us": "gpu__time_duration.sum",
    "dmma_active_pct": "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "shared_pipe_pct": "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "regs": "launch__registers_per_thread",
    "stall_wait": "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "stall_math_throttle": "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "stall_barrier": "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "stall_short_sb": "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "stall_long_sb": "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}

out = {}
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_summary.json")
if os.path.exists(path):
    out = json.load(open(path))
for arg in sys.argv[1:]:
    name, rep = arg.split("=", 1)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    kern = []
    for r in rows[2:]:
        e = {"kernel": r[hdr.index("Kernel Name")].split("(")[0][-70:], "grid": r[hdr.index("Grid Size")]}
        for k, m in KEYS.items():
            if m in hdr:
                i = hdr.index(m)
                v = float(r[i].replace(",", ""))
                u = units[i]
                if k in ("dram_read", "dram_write"):
                    v *= SCALE.get(u, 1)
                if k == "time_us":
                    v *= SCALE.get(u, 1)
                e[k] = round(v, 3)
        kern.append(e)
    gem = [k for k in kern if "gemm" in k["kernel"]]
    tb = sum(k["dram_read"] + k["dram_write"] for k in gem)
    out[name] = {"report": os.path.basename(rep), "launches": kern,
                 "gemm_dram_bytes_per_launch": tb / max(1, len(gem)),
                 "gemm_time_us_total": sum(k["time_us"] for k in gem)}
json.dump(out, open(path, "w"), indent=1)
print(json.dumps({k: (v["gemm_dram_bytes_per_launch"], v["gemm_time_us_total"]) for k, v in out.items()}))
