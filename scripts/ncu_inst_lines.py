"""Instructions executed and warp-stall samples per CUDA source line (cuda,sass source page)."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass",
                      "-k", kern, "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
res, fname, hdr = [], "", None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0]:
        continue
    try:
        res.append((int(r[7]), int(r[4] or 0), fname, r[0], r[1].strip()[:90]))
    except (ValueError, IndexError):
        pass
ti = sum(x[0] for x in res) or 1
ts = sum(x[1] for x in res) or 1
print(f"total warp instructions {ti}, stall samples {ts}")
for n, s, f, l, src in sorted(res, reverse=True)[:top]:
    print(f"{100 * n / ti:5.1f}% inst {100 * s / ts:5.1f}% stall  {f}:{l:>5s}  {src}")
