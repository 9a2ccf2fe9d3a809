"""Top SASS instructions by warp-stall samples (and executed counts) of one kernel in an ncu
report:  python tools/ncu_sass_hot.py report.ncu-rep [kernel-regex] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else "gemm"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", "regex:" + kern], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
    elif r and r[0] == "Address":
        cur["h"] = r
    elif cur is not None and "h" in cur and len(r) > 5:
        cur["rows"].append(r)
b = blocks[0]
h = b["h"]
iS, iE = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
data = [(float(r[iS] or 0), float(r[iE] or 0), i, r[1].strip()) for i, r in enumerate(b["rows"])]
tot = sum(d[0] for d in data)
tinst = sum(d[1] for d in data)
print(b["name"][:100], f"samples={tot:.0f} warp-inst={tinst:.0f}")
for s, n, i, src in sorted(data, reverse=True)[:top]:
    print(f"{s / tot * 100:5.1f}%  exec={n:9.0f}  #{i:5d}  {src[:90]}")
if len(sys.argv) > 4:
    # sample share per index range: argv[4] = "0-2000,2000-3400,3400-99999"
    for rg in sys.argv[4].split(","):
        a, z = map(int, rg.split("-"))
        s = sum(d[0] for d in data if a <= d[2] < z)
        n = sum(d[1] for d in data if a <= d[2] < z)
        print(f"range {rg}: {s / tot * 100:5.1f}% of samples, {n / tinst * 100:5.1f}% of warp-inst")
