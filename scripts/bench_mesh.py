"""Map export to a labelled mesh: extract_mesh on the device
(svx_mesh_extract) vs the reference's own extract_mesh (oracle/_ref, all host
threads) on the SAME map, with a full-size bit-exactness check of the two meshes.

Map: the cfg3 geometry (128-beam LiDAR, 0.05 m, tau 0.25 m, K = 20) plus the 6 label
images per frame, integrated on the GPU for FRAMES frames; the reference loads the
GPU map's SVOX1 snapshot (VoxelStore::load). Timed: the synchronous C-ABI call
(device) and extract + read back to host (e2e, what LabeledMesh users get).
Prints one JSON line."""
import json
import os
import sys
import tempfile
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("SEMVOX_THREADS", str(os.cpu_count() or 1))
import paper_2412_00291_b200 as svx  # noqa: E402
from paper_2412_00291_b200 import workload as W  # noqa: E402
from oracle import bindings as ob  # noqa: E402

FRAMES = int(os.environ.get("FRAMES", "40"))
REPS = int(os.environ.get("REPS", "10"))
REF_REPS = int(os.environ.get("REF_REPS", "2"))
wl = W.make(os.environ.get("WORKLOAD", "cfg3"), FRAMES)
cfg = svx.MapConfig(wl.voxel_size, wl.truncation, wl.num_labels, 1 << 22)
names = ["c%d" % k for k in range(wl.num_labels - 1)] + ["unlabeled"]

st = svx.VoxelStore(cfg, 0)
tsdf = svx.TsdfIntegrator(st, svx.IntegratorConfig())
sem = svx.SemanticIntegrator(st, svx.SemanticConfig())
t0 = time.time()
for p, i in wl.scans(device="cuda"):  # synthetic scans / label images rendered on the GPU
    tsdf.integrate_cloud(p.cpu().numpy(), wl.pose(i), wl.model)
    sem.integrate_labels_batch(wl.label_images(i, device="cuda"))
build_s = time.time() - t0
blocks = st.block_count()

lib = svx.lib()
h = st.handle
nv, nf = svx.C.c_uint64(), svx.C.c_uint64()


def extract():
    svx._check(lib.svx_mesh_extract(h, 1e-4, len(names) - 1, None, 0, svx.C.byref(nv),
                                    svx.C.byref(nf)))


for _ in range(3):  # warm-up (buffer growth, table upload)
    extract()
torch.cuda.synchronize()
dev_ms = []
for _ in range(REPS):
    t = time.perf_counter()
    extract()
    dev_ms.append(1e3 * (time.perf_counter() - t))
e2e_ms = []
for _ in range(REPS):
    t = time.perf_counter()
    mg = svx.extract_mesh(st, 1e-4, names)
    e2e_ms.append(1e3 * (time.perf_counter() - t))
V, F = mg.vertex_count(), int(mg.faces.shape[0])

out = {"metric": "mesh extraction (extract_mesh) ms per full-map export", "workload":
       f"{wl.name}: {FRAMES} frames (LiDAR + {len(wl.cams)} label images each), map of {blocks} "
       f"blocks", "blocks": blocks, "vertices": V, "faces": F,
       "device_ms": float(np.median(dev_ms)), "e2e_ms": float(np.median(e2e_ms)),
       "vertices_per_s": V / (np.median(e2e_ms) * 1e-3), "map_build_s": build_s}
# algorithmic bytes: the TSDF pool read once (20 B/voxel), both endpoint voxels +
# their K probabilities per vertex, the output (25 B/vertex + 12 B/face)
alg = blocks * 512 * 20 + V * (2 * 20 + 2 * 4 * wl.num_labels + 25) + F * 12
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
peak = float(peaks.get("hbm_gbs", 7672.0))
ach = alg / (out["device_ms"] * 1e-3) / 1e9
out["roofline"] = {"bound": "hbm", "alg_bytes": alg, "achieved": ach, "peak": peak, "unit": "GB/s",
                   "frac": ach / peak}

if ob.ref_available() and REF_REPS > 0:
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "map.svox")
        st.save(path)
        ref = ob.RefMap.load(path, cfg)
        ref_ms = []
        for _ in range(REF_REPS):
            t = time.perf_counter()
            mr = ref.extract_mesh(1e-4, len(names) - 1)
            ref_ms.append(1e3 * (time.perf_counter() - t))
        got = (mg.vertices, mg.vertex_normals, mg.vertex_labels, mg.faces)
        same = all(a.shape == b.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8))
                   for a, b in zip(got, mr))
        out["cpu_baseline"] = {"ms": float(np.median(ref_ms)), "cores": int(os.environ["SEMVOX_THREADS"]),
                               "kind": "reference", "sample": "the same map, whole-map extract_mesh "
                               "(reference mesh.cpp through oracle/_ref, parallel_for over blocks)"}
        out["speedup_e2e"] = float(np.median(ref_ms) / np.median(e2e_ms))
        out["bit_exact_vs_reference"] = bool(same)
print(json.dumps(out))
