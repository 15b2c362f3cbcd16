"""Per-frame store, then a batched store in the same process (test_batched_paths repro)."""
import os
import sys

import numpy as np
if not os.environ.get('SVXFIRST'):
    import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if os.environ.get("ORACLE"):
    from oracle import bindings as ob  # noqa: F401
    if os.environ.get("ORACLE") == "2":
        ob.OracleMap(ob.svx.MapConfig(0.1, 0.5, 2, 1024)) if hasattr(ob, "svx") else None
import paper_2412_00291_b200 as svx  # noqa: E402
from paper_2412_00291_b200 import workload as W  # noqa: E402

if os.environ.get('SVXFIRST'):
    import torch
wl = W.make("cfg2", int(sys.argv[1]) if len(sys.argv) > 1 else 12)
scans = [p.numpy() for p, _ in wl.scans()]
poses = [wl.pose(i) for i in range(len(scans))]
offs = np.zeros(len(scans) + 1, np.uint64)
offs[1:] = np.cumsum([s.shape[0] for s in scans])
flat = np.ascontiguousarray(np.concatenate(scans).astype(np.float32))
cfg = svx.MapConfig(wl.voxel_size, wl.truncation, wl.num_labels, 1 << 20)
ref = svx.VoxelStore(cfg, 0)
ti = svx.TsdfIntegrator(ref, svx.IntegratorConfig())
want = [ti.integrate_cloud(s, p, wl.model) for s, p in zip(scans, poses)]
print("per-frame ok", flush=True)
if os.environ.get("SAVE"):
    want_map = ref.save_bytes()
if os.environ.get("DIRTY"):
    want_dirty = np.asarray(ref.take_dirty_blocks(0))
dev = torch.from_numpy(flat).cuda()
if os.environ.get("PIN"):
    host = torch.from_numpy(flat).pin_memory()
if len(sys.argv) > 2:
    torch.cuda.synchronize()
st = svx.VoxelStore(cfg, 0)
if os.environ.get("PROF"):
    st.profile_enable(True)
got = st.integrate_clouds_device(wl.model, dev.data_ptr(), offs, 3, poses, svx.IntegratorConfig())
print("batched", all((a.updated_voxels, a.new_blocks) == (b.updated_voxels, b.new_blocks)
                     for a, b in zip(got, want)), st.save_bytes() == ref.save_bytes())
