"""Runs scripts/host_overhead.py against alternative builds (SVX_LIB) and prints
the mean per-frame kernel-group times of batches 2..N (kernel-variant A/B tests)."""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for lib in sys.argv[1:]:
    env = dict(os.environ)
    if lib != "default":
        env["SVX_LIB"] = os.path.abspath(lib)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "host_overhead.py")], env=env,
                         capture_output=True, text=True, timeout=600).stdout
    rows = [ln for ln in out.splitlines() if ln.startswith("prof=")][2:]
    acc, ev = {}, []
    for ln in rows:
        ev.append(float(re.search(r"events ([\d.]+)", ln).group(1)))
        for k, v in re.findall(r"(\w+)=([\d.]+)", ln.split("[")[1].split("]")[0]):
            acc.setdefault(k, []).append(float(v))
    med = sorted(ev)[len(ev) // 2] if ev else 0.0
    print(f"{lib:40s} events(median) {med:6.1f} us/frame  " +
          " ".join(f"{k}={sum(v) / len(v):.1f}" for k, v in acc.items()), flush=True)
