"""Batched-path repro: device / host batches, optionally with tiny buffers (env)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2412_00291_b200 as svx  # noqa: E402
from paper_2412_00291_b200 import workload as W  # noqa: E402

how = sys.argv[1]
nf = int(sys.argv[2]) if len(sys.argv) > 2 else 12
wl = W.make("cfg2", nf)
scans = [p.numpy() for p, _ in wl.scans()]
poses = [wl.pose(i) for i in range(len(scans))]
offs = np.zeros(len(scans) + 1, np.uint64)
offs[1:] = np.cumsum([s.shape[0] for s in scans])
flat = np.ascontiguousarray(np.concatenate(scans).astype(np.float32))
cfg = svx.MapConfig(wl.voxel_size, wl.truncation, wl.num_labels, 1 << 20)
st = svx.VoxelStore(cfg, 0)
st.profile_enable(True)
if how == "device":
    dev = torch.from_numpy(flat).cuda()
    got = st.integrate_clouds_device(wl.model, dev.data_ptr(), offs, 3, poses, svx.IntegratorConfig())
else:
    host = torch.from_numpy(flat).pin_memory()
    got = st.integrate_clouds_host(wl.model, host.data_ptr(), offs, 3, poses, svx.IntegratorConfig())
print(how, [(r.frame, r.updated_voxels, r.new_blocks) for r in got][:3], st.profile_read().as_dict()["aborts"])
