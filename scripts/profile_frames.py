"""Profiling driver: integrates `warm` cfg2 frames, then `frames` more inside a
cudaProfilerStart/Stop range (for `ncu --profile-from-start off`).

python scripts/profile_frames.py [workload] [warm] [frames]
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2412_00291_b200 as svx  # noqa: E402
from paper_2412_00291_b200 import workload as W  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    warm = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    frames = int(sys.argv[3]) if len(sys.argv) > 3 else 10
    wl = W.make(name, warm + frames)
    dev = torch.device("cuda", 0)
    chunks = [p for p, _ in wl.scans(device=dev)]
    counts = [c.shape[0] for c in chunks]
    pts = torch.cat(chunks).contiguous()
    offs = np.zeros(len(chunks) + 1, np.uint64)
    offs[1:] = np.cumsum(counts)
    cfg = svx.MapConfig(wl.voxel_size, wl.truncation, wl.num_labels, 1 << 21)
    s = svx.VoxelStore(cfg, 0)
    icfg = svx.IntegratorConfig()
    poses = [wl.pose(i) for i in range(len(chunks))]
    s.integrate_clouds_device(wl.model, pts.data_ptr(), offs[:warm + 1], 3, poses[:warm], icfg)
    torch.cuda.synchronize()
    s.profile_enable(True)
    torch.cuda.profiler.start()
    t0 = time.time()
    reps = s.integrate_clouds_device(wl.model, pts.data_ptr() + int(offs[warm]) * 12,
                                     offs[warm:] - offs[warm], 3, poses[warm:], icfg)
    torch.cuda.synchronize()
    t1 = time.time()
    torch.cuda.profiler.stop()
    p = s.profile_read().as_dict()
    print(f"{frames} frames in {(t1 - t0) * 1e3:.2f} ms wall; "
          f"{sum(counts[warm:]) / (t1 - t0) / 1e6:.1f} Mpts/s; upd/frame "
          f"{np.mean([r.updated_voxels for r in reps]):.0f}")
    print({k: round(v / frames * 1e3, 1) for k, v in p["ms"].items()}, "us/frame")
    print({k: p[k] for k in ("touched_blocks", "updated_voxels", "fallback_voxels", "rays")})


if __name__ == "__main__":
    main()
