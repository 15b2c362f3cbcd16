"""Generates tests/golden/seq_small.npz from the REFERENCE ITSELF.

Runs the reference's own translation units (oracle/_ref/libsemvox_ref.so, built
from /root/reference by oracle/Makefile) on a small fixed scan sequence and
stores inputs + outputs as fixtures, so the GPU path and the C restatement are
pinned to reference outputs even where /root/reference does not exist (GPU box).

    python tests/golden/make_golden.py          # needs oracle/_ref built here
"""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import paper_2412_00291_b200 as svx  # noqa: E402
from paper_2412_00291_b200 import workload as W  # noqa: E402
from oracle.bindings import RefMap, parse_svox1  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "seq_small.npz")


def main():
    model = svx.ProjectionModel.spinning(192, 24, 22.5, 22.5)
    scene = W.street_canyon(60.0, seed=7)
    poses = W.trajectory(3, 0.7, 1.73)
    g = __import__("torch").Generator()
    g.manual_seed(5)
    pts = [W.render_scan(scene, model, R, t, 0.02, g).numpy() for R, t in poses]
    cams = [(W._forward_cam(0.0), np.zeros(3), 96, 64, 48.0, 48.0, 48.0, 32.0)]
    wl = W.Workload("golden", model, 0.1, 0.5, 5, poses, scene, cams=cams)
    labels = []
    for i in range(len(poses)):
        for li in wl.label_images(i, seed=3, flip_rate=0.2):
            li.labels = (li.labels % 5).astype(np.uint16)
            labels.append(li)
    cfg = svx.MapConfig(0.1, 0.5, 5, 1 << 16)
    res = {}
    for mode in (svx.NON_PROJECTIVE, svx.PROJECTIVE):
        ref = RefMap(cfg)
        reps = []
        for i, (R, t) in enumerate(poses):
            pose = svx.pose_c(R, t)
            d, h, n, v, dr = RefMap.project(model, pts[i], pose)
            r = ref.integrate(model, d, n, v, pose, svx.IntegratorConfig(mode=mode))
            s = ref.integrate_labels(labels[i], svx.SemanticConfig())
            reps.append((r.updated_voxels, r.new_blocks, s.updated_voxels))
            if mode == svx.NON_PROJECTIVE:
                res[f"depth{i}"], res[f"height{i}"], res[f"normals{i}"], res[f"valid{i}"] = d, h, n, v
                res[f"dropped{i}"] = np.array(dr)
        blob = ref.save_bytes()
        hdr, keys, tsdf, sem = parse_svox1(blob)
        res[f"svox1_sha256_m{mode}"] = np.frombuffer(hashlib.sha256(blob).digest(), np.uint8)
        res[f"svox1_len_m{mode}"] = np.array(len(blob))
        res[f"reports_m{mode}"] = np.array(reps, np.int64)
        res[f"keys_m{mode}"] = keys
        res[f"observed_m{mode}"] = (tsdf["weight"] > 0).sum(axis=1).astype(np.int32)
        res[f"wsum_m{mode}"] = tsdf["weight"].astype(np.float64).sum(axis=1)
        res[f"sem_blocks_m{mode}"] = np.array(sorted(sem), np.int64)
    for i in range(len(poses)):
        res[f"points{i}"] = pts[i]
        res[f"pose{i}"] = np.concatenate([np.asarray(poses[i][0]).reshape(9), poses[i][1]])
        res[f"labels{i}"] = labels[i].labels
        res[f"cam_pose{i}"] = np.concatenate([np.array(labels[i].pose.R), np.array(labels[i].pose.t)])
    res["model"] = np.array([model.width, model.height_px, 22.5, 22.5])
    res["cam"] = np.array([96, 64, 48.0, 48.0, 48.0, 32.0, labels[0].max_depth])
    np.savez_compressed(OUT, **res)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
