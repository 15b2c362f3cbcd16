import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2412_00291_b200 as svx
from paper_2412_00291_b200 import workload as W
"""The batched entry points (clouds resident in HBM; clouds in pinned host memory,
staged through the ingest ring) produce the same map, reports and dirty lists as
one call per frame."""
import torch
wl = W.make("cfg2", 12)
scans = [p.numpy() for p, _ in wl.scans()]
poses = [wl.pose(i) for i in range(len(scans))]
offs = np.zeros(len(scans) + 1, np.uint64)
offs[1:] = np.cumsum([s.shape[0] for s in scans])
flat = np.ascontiguousarray(np.concatenate(scans).astype(np.float32))
cfg = svx.MapConfig(wl.voxel_size, wl.truncation, wl.num_labels, 1 << 20)
icfg = svx.IntegratorConfig()

ref = svx.VoxelStore(cfg, 0)
ti = svx.TsdfIntegrator(ref, icfg)
want = [ti.integrate_cloud(s, p, wl.model) for s, p in zip(scans, poses)]
want_map = ref.save_bytes()
want_dirty = np.asarray(ref.take_dirty_blocks(0))
assert len(want_dirty) > 1000

dev = torch.from_numpy(flat).cuda()
host = torch.from_numpy(flat).pin_memory()
import os
for how in os.environ.get("HOW", "device,host,host_split,device_resume").split(","):
    if how == "device_resume":  # tiny record buffer and pool headroom: abort + resume
        os.environ["SVX_TEST_REC_CAP"], os.environ["SVX_TEST_POOL_HEAD"] = "256", "16"
    try:
        st = svx.VoxelStore(cfg, 0)
    finally:
        os.environ.pop("SVX_TEST_REC_CAP", None)
        os.environ.pop("SVX_TEST_POOL_HEAD", None)
    if not os.environ.get('NOPROF'):
        st.profile_enable(True)
    if how.startswith("device"):
        got = st.integrate_clouds_device(wl.model, dev.data_ptr(), offs, 3, poses, icfg)
    elif how == "host":
        got = st.integrate_clouds_host(wl.model, host.data_ptr(), offs, 3, poses, icfg)
    else:  # two calls: frame numbering and state continue across batches
        got = st.integrate_clouds_host(wl.model, host.data_ptr(), offs[:6], 3, poses[:5], icfg)
        got += st.integrate_clouds_host(wl.model, host.data_ptr(), offs[5:], 3, poses[5:], icfg)
    assert [(r.frame, r.updated_voxels, r.new_blocks) for r in got] == \
        [(r.frame, r.updated_voxels, r.new_blocks) for r in want], how
    assert st.save_bytes() == want_map, how
    assert np.array_equal(np.asarray(st.take_dirty_blocks(0)), want_dirty), how
    aborts = st.profile_read().as_dict()["aborts"]
    if how == "device_resume":
        assert aborts.get("records", 0) >= 1, aborts
    st.close()
ref.close()
