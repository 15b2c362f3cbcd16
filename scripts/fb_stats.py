import sys, json, numpy as np, torch
sys.path.insert(0, '.')
import paper_2412_00291_b200 as svx
from paper_2412_00291_b200 import workload as W
dev = torch.device('cuda', 0)
for Wd in [int(x) for x in sys.argv[1:]]:
    n = 16
    wl = W.make(f"cfg5-{Wd}", 3 * n + 8)
    chunks = [p for p, _ in wl.scans(device=dev)]
    offs = np.zeros(len(chunks) + 1, np.uint64); offs[1:] = np.cumsum([c.shape[0] for c in chunks])
    pts = torch.cat(chunks).contiguous()
    poses = [wl.pose(i) for i in range(len(chunks))]
    st = svx.VoxelStore(svx.MapConfig(wl.voxel_size, wl.truncation, wl.num_labels, 1 << 21), 0)
    icfg = svx.IntegratorConfig()
    for first in (0, 8, 8 + n):
        if first == 8 + n: st.profile_enable(True)
        cnt = n if first else 8
        rel = offs[first:first + cnt + 1] - offs[first]
        torch.cuda.synchronize()
        reps = st.integrate_clouds_device(wl.model, pts.data_ptr() + 12 * int(offs[first]), rel, 3, poses[first:first + cnt], icfg)
    p = st.profile_read().as_dict()
    print(json.dumps({"W": Wd, **{k: v for k, v in p.items()}}), flush=True)
    st.close()
