"""Top SASS instructions by warp-stall samples from an ncu report (source page)."""
import csv
import subprocess
import sys
from collections import Counter

rep, kern = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
args = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"]
out = subprocess.run(args, capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
# the page holds one table per profiled kernel: "Kernel Name" row, header row, data
tables, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        tables.append(cur)
    elif cur is not None:
        cur["rows"].append(r)
tab = next(t for t in tables if kern in t["name"])
hdr = tab["rows"][0]
data = [dict(zip(hdr, r)) for r in tab["rows"][1:] if len(r) == len(hdr)]
tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
stalls = Counter()
for d in data:
    for k, v in d.items():
        if k.startswith("stall_") and "Not Issued" not in k:
            try:
                stalls[k] += int(v)
            except ValueError:
                pass
print("total samples", tot)
print("stall mix:", ", ".join(f"{k[6:]}={100*v/tot:.1f}%" for k, v in stalls.most_common(8)))
ops = Counter()
for d in data:
    op = d["Source"].split()[0] if d["Source"].split() else "?"
    if op.startswith("@"):
        op = d["Source"].split()[1]
    ops[op.split(".")[0]] += int(d["Warp Stall Sampling (All Samples)"] or 0)
print("by opcode:", ", ".join(f"{k}={100*v/tot:.1f}%" for k, v in ops.most_common(14)))
idx = sorted(range(len(data)), key=lambda i: -int(data[i]["Warp Stall Sampling (All Samples)"] or 0))
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
for i in idx[:n]:
    d = data[i]
    s = int(d["Warp Stall Sampling (All Samples)"] or 0)
    top = max(((int(v or 0), k) for k, v in d.items() if k.startswith("stall_") and "Not" not in k and v.isdigit()), default=(0, ""))
    print(f"{100*s/tot:5.1f}% [{i:5d}] {d['Source'][:70]:70s} thr={d['Avg. Threads Executed']} {top[1][6:]}")
