"""Aggregate an ncu --metrics gpu__time_duration.sum CSV launch list per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    k = d["Kernel Name"].split("(")[0].split("::")[-1]
    unit = d.get("Metric Unit", "ns")
    v = float(d["Metric Value"].replace(",", ""))
    v = v * (1e3 if unit == "us" else 1e6 if unit == "ms" else 1.0)  # -> ns
    agg[k][0] += 1
    agg[k][1] += v
total = sum(t for _, t in agg.values())
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 1
print(f"{'kernel':28s} {'n':>5s} {'us/frame':>9s} {'avg us':>8s} {'share':>6s}")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:28s} {n:5d} {t / 1e3 / frames:9.1f} {t / n / 1e3:8.2f} {100 * t / total:5.1f}%")
print(f"{'total':28s} {'':5s} {total / 1e3 / frames:9.1f}")
