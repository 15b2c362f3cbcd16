"""Per-call timing of the exchange-mode calls (xbegin / xend) for N ranks emulated on
one GPU: host wall time vs device time (CUDA events on the map stream)."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2412_00291_b200 as svx  # noqa: E402
from paper_2412_00291_b200 import dist as sdist  # noqa: E402
from paper_2412_00291_b200 import workload as W  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 4
frames = 160
wl = W.make("cfg2", frames)
dev = torch.device("cuda", 0)
chunks = [p for p, _ in wl.scans(device=dev)]
offs = np.zeros(frames + 1, np.uint64)
offs[1:] = np.cumsum([c.shape[0] for c in chunks])
pts = torch.cat(chunks).contiguous()
poses = [wl.pose(i) for i in range(frames)]
cfg = svx.MapConfig(wl.voxel_size, wl.truncation, wl.num_labels, 1 << 21)
icfg = svx.IntegratorConfig()
stores = []
for r in range(N):
    st = svx.VoxelStore(cfg, 0)
    st.set_shard(r, N)
    stores.append(st)
rows = []
stores[0].profile_enable(True)
for a in range(0, frames, 16):
    rel = offs[a:a + 17] - offs[a]
    sends, counts, tb, db = [], [], [], []
    for st in stores:
        ext = torch.cuda.ExternalStream(st.stream_ptr(), device=dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(ext)
        t0 = time.perf_counter()
        c, ptr = st.xbegin(wl.model, pts.data_ptr() + int(offs[a]) * 12, rel, 3, poses[a:a + 16], icfg)
        c = c.astype(np.int64)
        tb.append((time.perf_counter() - t0) * 1e3)
        e1.record(ext)
        e1.synchronize()
        db.append(e0.elapsed_time(e1))
        sends.append(sdist.device_bytes(ptr, int(c[:, 0].sum()) * 16, dev).clone())
        counts.append(c)
    te, de = [], []
    for d, st in enumerate(stores):
        parts = [sends[r][int(counts[r][:d, 0].sum()) * 16:int(counts[r][:d + 1, 0].sum()) * 16] for r in range(N)]
        recv = torch.cat(parts)
        rmeta = np.stack([counts[r][d] for r in range(N)])
        ext = torch.cuda.ExternalStream(st.stream_ptr(), device=dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(ext)
        t0 = time.perf_counter()
        st.xend(recv.data_ptr(), rmeta)
        te.append((time.perf_counter() - t0) * 1e3)
        e1.record(ext)
        e1.synchronize()
        de.append(e0.elapsed_time(e1))
    if a >= 64:
        rows.append({"xbegin_wall": max(tb), "xbegin_dev": max(db), "xend_wall": max(te), "xend_dev": max(de),
                     "entries": int(sum(c[:, 0].sum() for c in counts))})
prof = stores[0].profile_read().as_dict()
print(json.dumps({"N": N, "per_group_ms": {k: float(np.mean([r[k] for r in rows])) for k in rows[0]},
                  "rank0_kernel_ms_per_group": {k: v / (frames / 16) for k, v in prof["ms"].items()},
                  "host_ms": {k: prof[k] for k in ("host_enqueue_ms", "host_map_ms")}}))
