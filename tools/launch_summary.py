"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
    python tools/launch_summary.py <launches.csv> "<command line>" > profiles/<name>.txt"""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if "Kernel Name" in r)
agg = collections.OrderedDict()
for r in rows[rows.index(hdr) + 1:]:
    if len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(d["Metric Value"].replace(",", ""))
    v = v / 1e3 if d["Metric Unit"] == "ns" else v * 1e3 if d["Metric Unit"] == "ms" else v
    k = d["Kernel Name"][:80]
    n, t = agg.get(k, (0, 0.0))
    agg[k] = (n + 1, t + v)
print("ncu --metrics gpu__time_duration.sum --clock-control none (cold, serialised) launch list of")
print("  " + (sys.argv[2] if len(sys.argv) > 2 else ""))
tot = sum(t for _, t in agg.values())
for k, (n, t) in agg.items():
    print(f"  {n:3d} x {t / n:10.1f} us  {100 * t / tot:5.1f}%  {k}")
