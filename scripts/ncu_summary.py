"""Summarise an ncu report: per-kernel duration, throughput, occupancy, pipes, stalls, DRAM bytes.

usage: ncu_summary.py REPORT [JSON_OUT] [G]   (JSON_OUT: per-kernel mean duration and DRAM
bytes per launch, read by bench.py for the roofline `traffic` field; G = frames per launch
of the frame-group kernels (k_fold runs once per frame))"""
import csv
import json
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
json_out = sys.argv[2] if len(sys.argv) > 2 else None
group = int(sys.argv[3]) if len(sys.argv) > 3 else 1
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
want = {
    "gpu__time_duration.sum": "dur",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm%",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem%",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occ%",
    "smsp__inst_executed.sum": "inst",
    "launch__registers_per_thread": "regs",
    "lts__t_sector_hit_rate.pct": "l2hit%",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64%",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu%",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma%",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu%",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu%",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "thr/warp",
}
stall = "smsp__average_warps_issue_stalled_"
scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "ms": 1e3,
         "usecond": 1.0, "nsecond": 1e-3, "msecond": 1e3}
agg = defaultdict(lambda: {"launches": 0, "us": 0.0, "dram_bytes": 0.0})


def num(d, k):
    u = units[hdr.index(k)]
    return float(d[k].replace(",", "")) * scale.get(u, 1.0)


for r in rows[2:]:
    d = dict(zip(hdr, r))
    name = d["Kernel Name"].split("(")[0].split("::")[-1]
    out = []
    for k, lab in want.items():
        if k in d:
            out.append(f"{lab}={d[k]}{units[hdr.index(k)]}")
    st = []
    for h, v in d.items():
        if h.startswith(stall) and h.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(v), h[len(stall):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    st.sort(reverse=True)
    a = agg[name]
    a["launches"] += 1
    a["us"] += num(d, "gpu__time_duration.sum")
    a["dram_bytes"] += num(d, "dram__bytes_read.sum") + num(d, "dram__bytes_write.sum")
    print(f"== {name}: " + " ".join(out))
    print("   stalls(top): " + ", ".join(f"{n}={v:.1f}" for v, n in st[:6]))

if json_out:
    res = {k: {"launches": v["launches"], "us_per_launch": v["us"] / v["launches"],
               "dram_bytes_per_launch": v["dram_bytes"] / v["launches"],
               "frames_per_launch": 1 if k == "k_fold" else group} for k, v in agg.items()}
    json.dump({"report": rep.split("/")[-1], "kernels": res}, open(json_out, "w"), indent=1)
