"""Summarise an ncu --csv launch list (gpu__time_duration + optional DMMA %) per kernel."""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi, mi, gi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Value", "Metric Name", "Grid Size", "ID"))
d = {}
for r in rows[1:]:
    e = d.setdefault(r[ii], {})
    e[r[mi]] = r[vi]
    e["k"], e["g"] = r[ki], r[gi]
tot = 0.0
for v in d.values():
    t = float(v["gpu__time_duration.sum"].replace(",", "")) / 1000
    tot += t
    dm = v.get("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "")
    name = v["k"].split("(")[0].replace("void (anonymous namespace)::", "").replace("void unnamed>::", "")
    print(f"{t:9.1f} us  dmma {dm[:5]:>5s}  grid {v['g']:14s} {name[:80]}")
print(f"total {tot:.1f} us over {len(d)} launches")
