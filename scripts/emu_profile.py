"""Per-rank kernel breakdown of the exchange-mode data plane with N ranks emulated on one
GPU (dist.emulate_sharded): where a rank's time goes as N grows.
Usage: python scripts/emu_profile.py [N ...]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_00291_b200 as svx  # noqa: E402
from paper_2412_00291_b200 import dist as sdist  # noqa: E402
from paper_2412_00291_b200 import workload as W  # noqa: E402

dev = torch.device("cuda", 0)
spp, steps, warm = 96, 2, 1
n_frames = (steps + warm) * spp
wl = W.make("cfg2", n_frames)
chunks = [p for p, _ in wl.scans(device=dev)]
offs = np.zeros(n_frames + 1, np.uint64)
offs[1:] = np.cumsum([c.shape[0] for c in chunks])
pts = torch.cat(chunks).contiguous()
poses = [wl.pose(i) for i in range(n_frames)]
cfg = svx.MapConfig(wl.voxel_size, wl.truncation, wl.num_labels, 1 << 21)
icfg = svx.IntegratorConfig()
for N in [int(a) for a in sys.argv[1:]] or [1, 8]:
    stores = []
    for r in range(N):
        st = svx.VoxelStore(cfg, 0)
        st.reserve(1 << 18)
        if N > 1:
            st.set_shard(r, N)
        stores.append(st)
    step_ms = []
    for s in range(warm + steps):
        if s == warm:
            for st in stores:
                st.profile_read()
                st.profile_enable(True)
        f0, f1 = s * spp, (s + 1) * spp
        rel = offs[f0:f1 + 1] - offs[f0]
        timers = []
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if N > 1:
            sdist.emulate_sharded(stores, wl.model, pts.data_ptr() + int(offs[f0]) * 12, rel, 3, poses[f0:f1], icfg,
                                  timers=timers)
        else:
            stores[0].integrate_clouds_device(wl.model, pts.data_ptr() + int(offs[f0]) * 12, rel, 3, poses[f0:f1], icfg)
        torch.cuda.synchronize()
        step_ms.append(round((time.perf_counter() - t0) * 1e3, 2))
    print(json.dumps({"N": N, "step_ms": step_ms}), flush=True)
    for r, st in enumerate(stores[:2]):
        p = st.profile_read().as_dict()
        print(json.dumps({"N": N, "rank": r, "us_per_frame": {k: round(1e3 * v / (steps * spp), 2) for k, v in p["ms"].items()},
                          "launches": p["launches"], "host_enqueue_ms": p["host_enqueue_ms"],
                          "host_resume_ms": p["host_resume_ms"], "host_map_ms": p["host_map_ms"],
                          "aborts": p["aborts"]}), flush=True)
    for st in stores:
        st.close()
