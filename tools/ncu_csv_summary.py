"""Per-kernel mean of each metric in an `ncu --csv` launch list: python tools/ncu_csv_summary.py F.csv ..."""
import collections
import csv
import sys

for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    h = next((i for i, r in enumerate(rows) if "Kernel Name" in r and "Metric Name" in r), None)
    if h is None:
        print(path, "no ncu rows")
        continue
    hdr = rows[h]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[h + 1:]:
        if len(r) > vi:
            agg[(r[ki].split("(")[0][-40:], r[mi])].append(float(r[vi].replace(",", "")))
    print(path)
    for (k, m), v in sorted(agg.items()):
        print(f"  {k:40s} {m:28s} n={len(v):3d} mean={sum(v) / len(v):.4g}")
