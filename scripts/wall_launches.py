"""Per-kernel totals and the longest launches from an ncu launch list (csv, gpu__time_duration.sum)."""
import collections
import csv
import sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, out = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            out.append((int(d["ID"]), d["Kernel Name"].split("(")[0].split("::")[-1], float(d["Metric Value"].replace(",", ""))))
tot, cnt = collections.Counter(), collections.Counter()
for _, k, t in out:
    tot[k] += t
    cnt[k] += 1
for k, t in tot.most_common():
    print("%-16s n=%4d total %.2f ms max %.3f ms" % (k, cnt[k], t / 1e6, max(x[2] for x in out if x[1] == k) / 1e6))
