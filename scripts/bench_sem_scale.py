"""Semantic pass cost vs map size: cfg4 city trajectory, geometry for
4000 scans; every 400 scans one frame's label image is integrated and the semantic kernel
times (frustum cull over the device block list, fused update) are recorded against the
number of allocated blocks. The cull reads 8 B per block (key) plus a distance test; the
update touches only frustum candidates."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2412_00291_b200 as svx  # noqa: E402
from paper_2412_00291_b200 import workload as W  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
every = 400
wl = W.make("cfg4", n)
dev = torch.device("cuda", 0)
cfg = svx.MapConfig(wl.voxel_size, wl.truncation, wl.num_labels, 1 << 22)
st = svx.VoxelStore(cfg, 0)
si = svx.SemanticIntegrator(st)
icfg = svx.IntegratorConfig()
rows = []
for a in range(0, n, every):
    frames = list(range(a, min(n, a + every)))
    chunks = [p for p, _ in wl.scans(device=dev, frames=frames)]
    offs = np.zeros(len(chunks) + 1, np.uint64)
    offs[1:] = np.cumsum([c.shape[0] for c in chunks])
    pts = torch.cat(chunks).contiguous()
    st.integrate_clouds_device(wl.model, pts.data_ptr(), offs, 3, [wl.pose(i) for i in frames], icfg)
    imgs = wl.label_images(frames[-1], device=dev)
    dimgs = [svx.LabelImage(li.width, li.height, torch.from_numpy(np.asarray(li.labels).view(np.int16).copy()).to(dev),
                            li.fx, li.fy, li.cx, li.cy, li.pose, max_depth=li.max_depth) for li in imgs]
    torch.cuda.synchronize()
    si.integrate_labels_batch(dimgs, on_device=True)  # warm
    st.profile_enable(True)
    reps = si.integrate_labels_batch(dimgs, on_device=True)
    p = st.profile_read().as_dict()
    st.profile_enable(False)
    rows.append({"frame": frames[-1], "blocks": st.block_count(), "updated": sum(r.updated_voxels for r in reps),
                 "candidates": p["sem_candidates"], "cull_us": 1e3 * p["ms"].get("sem_cull", 0.0),
                 "update_us": 1e3 * p["ms"].get("sem_update", 0.0)})
    print(json.dumps(rows[-1]), flush=True)
print(json.dumps({"semantic_scale": rows}))
