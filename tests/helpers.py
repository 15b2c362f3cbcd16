"""Shared test helpers: golden fixture access and map comparison."""
import hashlib
import os

import numpy as np

import paper_2412_00291_b200 as svx
from oracle.bindings import parse_svox1

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "seq_small.npz")


class Golden:
    def __init__(self):
        self.d = np.load(GOLDEN)
        w, h, up, down = self.d["model"]
        self.model = svx.ProjectionModel.spinning(int(w), int(h), float(up), float(down))
        self.cfg = svx.MapConfig(0.1, 0.5, 5, 1 << 16)
        self.n = 3

    def points(self, i):
        return self.d[f"points{i}"]

    def pose(self, i):
        p = self.d[f"pose{i}"]
        return svx.pose_c(p[:9].reshape(3, 3), p[9:])

    def label_image(self, i):
        W_, H_, fx, fy, cx, cy, md = self.d["cam"]
        cp = self.d[f"cam_pose{i}"]
        return svx.LabelImage(int(W_), int(H_), self.d[f"labels{i}"], fx, fy, cx, cy,
                              svx.pose_c(cp[:9].reshape(3, 3), cp[9:]), max_depth=md)

    def check_map(self, blob: bytes, mode: int):
        """Asserts a SVOX1 image equals the reference's (sha256), with diagnostics."""
        hdr, keys, tsdf, sem = parse_svox1(blob)
        assert np.array_equal(keys, self.d[f"keys_m{mode}"]), "allocated block set differs"
        assert np.array_equal((tsdf["weight"] > 0).sum(axis=1), self.d[f"observed_m{mode}"]), \
            "observed voxel set differs"
        assert np.array_equal(tsdf["weight"].astype(np.float64).sum(axis=1),
                              self.d[f"wsum_m{mode}"]), "weights differ"
        assert np.array_equal(np.array(sorted(sem)), self.d[f"sem_blocks_m{mode}"]), \
            "semantic-layer presence differs"
        assert len(blob) == int(self.d[f"svox1_len_m{mode}"])
        assert hashlib.sha256(blob).digest() == self.d[f"svox1_sha256_m{mode}"].tobytes(), \
            "SVOX1 bytes differ from the reference's snapshot"


def compare_maps(a: bytes, b: bytes, tol: float = 1e-5, exact: bool = False):
    """Parity contract: same block keys, observed set, W exact,
    semantic layers + probs exact, D and g within `tol`. Returns stats."""
    ha, ka, ta, sa = parse_svox1(a)
    hb, kb, tb, sb = parse_svox1(b)
    assert ha == hb
    assert np.array_equal(ka, kb), "block key sets differ"
    assert np.array_equal(ta["weight"] > 0, tb["weight"] > 0), "observed sets differ"
    assert np.array_equal(ta["weight"], tb["weight"]), "weights differ"
    dd = np.abs(ta["distance"] - tb["distance"]).max() if len(ka) else 0.0
    dg = np.abs(ta["gradient"] - tb["gradient"]).max() if len(ka) else 0.0
    assert dd <= tol and dg <= tol, (dd, dg)
    assert sorted(sa) == sorted(sb), "semantic layer presence differs"
    for k in sa:
        assert np.array_equal(sa[k], sb[k]), "semantic probabilities differ"
    if exact:
        assert a == b, "SVOX1 bytes differ"
    return {"blocks": len(ka), "d_max": float(dd), "g_max": float(dg), "bytes_equal": a == b}
