"""Warp-stall samples per CUDA source line (cuda,sass source page of an ncu report)."""
import csv
import subprocess
import sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass",
                      "-k", kern], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
per_line = defaultdict(int)
text = {}
fname = ""
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        hdr = None
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 5:
        continue
    line, src = r[0], r[1]
    if line:
        text[(fname, line)] = src
        try:
            per_line[(fname, line)] += int(r[4] or 0)
        except ValueError:
            pass
tot = sum(per_line.values()) or 1
for (f, l), v in sorted(per_line.items(), key=lambda x: -x[1])[:top]:
    print(f"{100 * v / tot:5.1f}% {f}:{l:>5s}  {text[(f, l)].strip()[:100]}")
