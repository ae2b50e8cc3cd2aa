"""Summarise an ncu --csv launch list (per kernel: launches, avg time, share, metric means)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[start]
ix = {k: h.index(k) for k in h}
agg = collections.OrderedDict()
for r in rows[start + 1:]:
    if len(r) < len(h):
        continue
    k = r[ix["Kernel Name"]][:48]
    # split identical kernel names by grid size (projection vs target-side launches of the same GEMM)
    k += " " + r[ix["Grid Size"]] if "Grid Size" in ix else ""
    v = float(r[ix["Metric Value"]].replace(",", ""))
    agg.setdefault(k, {}).setdefault(r[ix["Metric Name"]], []).append(v)
tot = sum(sum(v.get("gpu__time_duration.sum", [0])) for v in agg.values())
for k, v in agg.items():
    t = v.get("gpu__time_duration.sum", [0])
    extra = " ".join(f"{m.split('.')[0].split('__')[-1][:18]}={sum(x)/len(x):.3g}" for m, x in v.items() if m != "gpu__time_duration.sum")
    print(f"{k:64s} n={len(t):3d} avg={sum(t)/len(t)/1e3:9.1f}us share={sum(t)/tot*100:5.1f}% {extra}")
