"""Timeline of one emulated exchange-mode step (N ranks on one GPU, dist.emulate_sharded)
under torch.profiler (CUPTI): GPU busy vs idle time inside the step and the CUDA runtime
calls the host spends the most time in (where a rank's ~16 us of host time per frame goes,
DESIGN.md section 6). Usage: python scripts/emu_trace.py [N]"""
import collections
import json
import os
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_00291_b200 as svx  # noqa: E402
from paper_2412_00291_b200 import dist as sdist  # noqa: E402
from paper_2412_00291_b200 import workload as W  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
dev = torch.device("cuda", 0)
spp, warm = 96, 2
n_frames = (warm + 1) * spp
wl = W.make("cfg2", n_frames)
chunks = [p for p, _ in wl.scans(device=dev)]
offs = np.zeros(n_frames + 1, np.uint64)
offs[1:] = np.cumsum([c.shape[0] for c in chunks])
pts = torch.cat(chunks).contiguous()
poses = [wl.pose(i) for i in range(n_frames)]
cfg = svx.MapConfig(wl.voxel_size, wl.truncation, wl.num_labels, 1 << 21)
icfg = svx.IntegratorConfig()
stores = []
for r in range(N):
    st = svx.VoxelStore(cfg, 0)
    st.reserve(1 << 18)
    st.set_shard(r, N)
    stores.append(st)


def step(s, timers=None):
    f0, f1 = s * spp, (s + 1) * spp
    rel = offs[f0:f1 + 1] - offs[f0]
    sdist.emulate_sharded(stores, wl.model, pts.data_ptr() + int(offs[f0]) * 12, rel, 3, poses[f0:f1], icfg,
                          timers=timers)


for s in range(warm):
    step(s)
torch.cuda.synchronize()
timers = []
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    step(warm, timers)
    torch.cuda.synchronize()
ev = prof.events()
gpu = sorted([(e.time_range.start, e.time_range.end, e.name) for e in ev
              if e.device_type == torch.autograd.DeviceType.CUDA], key=lambda x: x[0])
t0, t1 = gpu[0][0], max(e[1] for e in gpu)
busy, cur_s, cur_e = 0.0, None, None
for a, b, _ in gpu:
    if cur_e is None or a > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = a, b
    else:
        cur_e = max(cur_e, b)
busy += cur_e - cur_s
api = collections.defaultdict(lambda: [0, 0.0])
for e in ev:
    if e.device_type == torch.autograd.DeviceType.CPU and e.name.startswith("cuda"):
        api[e.name][0] += 1
        api[e.name][1] += e.time_range.end - e.time_range.start
kern = collections.defaultdict(lambda: [0, 0.0])
for a, b, nm in gpu:
    kern[nm[:60]][0] += 1
    kern[nm[:60]][1] += b - a
rank_ms = sum(max(b + e for b, e in zip(t["xbegin_ms"], t["xend_ms"])) for t in timers)
all_ms = sum(sum(t["xbegin_ms"]) + sum(t["xend_ms"]) for t in timers)
print(json.dumps({"N": N, "frames": spp, "gpu_span_ms": (t1 - t0) / 1e3, "gpu_busy_ms": busy / 1e3,
                  "sum_rank_call_ms": all_ms, "max_rank_ms_under_profiler": rank_ms,
                  "api_top": sorted(([k, v[0], round(v[1] / 1e3, 3)] for k, v in api.items()),
                                    key=lambda x: -x[2])[:14],
                  "gpu_top": sorted(([k, v[0], round(v[1] / 1e3, 3)] for k, v in kern.items()),
                                    key=lambda x: -x[2])[:20]}, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
prof.export_chrome_trace(f"gpurun_out/emu_trace_n{N}.json")
