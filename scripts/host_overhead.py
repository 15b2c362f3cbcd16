"""Host vs device time of the batched frame path (profiling on/off)."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2412_00291_b200 as svx  # noqa: E402
from paper_2412_00291_b200 import workload as W  # noqa: E402

wl = W.make("cfg2", 1000)
dev = torch.device("cuda", 0)
chunks = [p for p, _ in wl.scans(device=dev)]
pts = torch.cat(chunks).contiguous()
offs = np.zeros(len(chunks) + 1, np.uint64)
offs[1:] = np.cumsum([c.shape[0] for c in chunks])
poses = [wl.pose(i) for i in range(len(chunks))]
cfg = svx.MapConfig(wl.voxel_size, wl.truncation, wl.num_labels, 1 << 21)
icfg = svx.IntegratorConfig()
s = svx.VoxelStore(cfg, 0)
ext = torch.cuda.ExternalStream(s.stream_ptr())
f = 0
for prof in (True,) * 10:
    s.profile_enable(prof)
    for batch in (100,):
        a, b = f, f + batch
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ext)
        t0 = time.perf_counter()
        s.integrate_clouds_device(wl.model, pts.data_ptr() + int(offs[a]) * 12, offs[a:b + 1] - offs[a],
                                  3, poses[a:b], icfg)
        t1 = time.perf_counter()
        e1.record(ext)
        e1.synchronize()
        p = s.profile_read().as_dict() if prof else {"ms": {}}
        ksum = sum(p["ms"].values())
        groups = " ".join(f"{k}={1e3 * v / batch:.1f}" for k, v in p["ms"].items())
        print(f"prof={prof} frames {a}-{b}: call {1e6 * (t1 - t0) / batch:.1f} us/frame, events "
              f"{1e3 * e0.elapsed_time(e1) / batch:.1f} us/frame, kernel groups {1e3 * ksum / batch:.1f}"
              f" us/frame [{groups}], host enqueue {1e3 * p.get('host_enqueue_ms', 0) / batch:.1f} us/frame,"
              f" blocks {s.block_count()} aborts {p.get('aborts')} resume {p.get('host_resume_ms', 0):.1f} ms map {p.get('host_map_ms', 0):.1f} ms")
        f = b
