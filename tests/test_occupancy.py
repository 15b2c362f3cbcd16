"""Occupancy extension (include/svx.h "occupancy extension"):
free-space carving, per-scan HIT/MISS dedup, log-odds, hit/miss counters, integer
class histograms. The reference has none of this (SPEC.md:255 declines carving), so
PARITY IS UNPINNED: the oracle (svxo_occ_*) restates the project's own contract and
is checked here against hand-derived known answers and the contract's properties
(order independence, hit dominance, clamping, range cut, capacity rejection); the
GPU must reproduce the oracle's SOCC1 export byte for byte."""
import numpy as np
import pytest

import paper_2412_00291_b200 as svx
from oracle import bindings as ob

needs_oracle = pytest.mark.skipif(not ob.oracle_available(), reason="oracle not built")


def occ_cfg(**kw):
    c = svx.OccupancyConfig(voxel_size=0.1, num_labels=4, max_blocks=1 << 12)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def voxel(parsed, v):
    """(L, hits, misses, hist row | None) of voxel v from a parsed SOCC1."""
    hdr, keys, L, hits, misses, hist = parsed
    b = np.floor_divide(np.asarray(v), 8)
    i = np.where(np.all(keys == b, axis=1))[0]
    if not len(i):
        return None
    i = int(i[0])
    lin = (v[0] & 7) + 8 * (v[1] & 7) + 64 * (v[2] & 7)
    return float(L[i, lin]), int(hits[i, lin]), int(misses[i, lin]), (hist[i][lin] if i in hist else None)


@needs_oracle
def test_single_ray_known_answer():
    o = ob.OracleOcc(occ_cfg())
    r = o.integrate(np.array([[1.0, 0, 0]], np.float32), svx.pose_c())
    assert (r.rays, r.hit_voxels, r.miss_voxels, r.new_blocks) == (1, 1, 10, 2)
    p = ob.parse_socc1(o.save_bytes())
    for x in range(10):  # world_to_voxel(1.0 / 0.1) = 10 is the hit voxel
        assert voxel(p, (x, 0, 0))[:3] == (np.float32(-0.4), 0, 1)
    assert voxel(p, (10, 0, 0))[:3] == (np.float32(0.85), 1, 0)
    assert voxel(p, (11, 0, 0))[:3] == (0.0, 0, 0)


@needs_oracle
def test_hit_dominates_and_once_per_scan():
    """Voxel 10 is hit by one ray and crossed by another: one HIT update; the
    crossed voxels are updated once although two rays cross them."""
    o = ob.OracleOcc(occ_cfg())
    pts = np.array([[1.0, 0, 0], [2.0, 0, 0]], np.float32)
    r = o.integrate(pts, svx.pose_c())
    assert (r.hit_voxels, r.miss_voxels) == (2, 19)  # misses 0-9, 11-19
    p = ob.parse_socc1(o.save_bytes())
    assert voxel(p, (10, 0, 0))[:3] == (np.float32(0.85), 1, 0)
    assert voxel(p, (5, 0, 0))[:3] == (np.float32(-0.4), 0, 1)


@needs_oracle
def test_clamping_and_counters_over_scans():
    o = ob.OracleOcc(occ_cfg())
    for _ in range(6):
        o.integrate(np.array([[1.0, 0, 0]], np.float32), svx.pose_c())
    p = ob.parse_socc1(o.save_bytes())
    L, h, m, _ = voxel(p, (10, 0, 0))
    assert (h, m) == (6, 0) and L == np.float32(3.5)      # 6 * 0.85 clamps at l_max
    L, h, m, _ = voxel(p, (3, 0, 0))
    assert (h, m) == (0, 6) and L == np.float32(-2.0)     # clamps at l_min


@needs_oracle
def test_max_range_cut_and_min_range_drop():
    o = ob.OracleOcc(occ_cfg(max_range=0.57))
    r = o.integrate(np.array([[1.0, 0, 0], [0.1, 0, 0], [np.nan, 0, 0]], np.float32), svx.pose_c())
    assert (r.points, r.rays, r.hit_voxels) == (3, 1, 0)  # 0.1 < min_range, NaN dropped
    p = ob.parse_socc1(o.save_bytes())
    assert voxel(p, (6, 0, 0))[:3] == (np.float32(-0.4), 0, 1)  # end cut at 0.57 -> voxel 6
    assert voxel(p, (7, 0, 0))[:3] == (0.0, 0, 0)


@needs_oracle
def test_histogram_fixed_point_and_argmax():
    o = ob.OracleOcc(occ_cfg(carve=False))
    pts = np.array([[1.0, 0, 0]] * 4, np.float32)
    o.integrate(pts, svx.pose_c(), labels=np.array([2, 1, 1, 9], np.uint16),
                conf=np.array([0.9, 0.5, 0.3, 1.0], np.float32))
    p = ob.parse_socc1(o.save_bytes())
    L, h, m, hist = voxel(p, (10, 0, 0))
    # q8 = (uint32)(c*255 + 0.5): 0.9 -> 230, 0.5 -> 128, 0.3 -> 77; label 9 >= K ignored
    assert list(hist) == [0, 128 + 77, 230, 0]
    assert (h, m) == (1, 0) and p[1].shape[0] == 1   # carve off: only the hit block


@needs_oracle
def test_order_independence():
    wl = __import__("paper_2412_00291_b200.workload", fromlist=["make"]).make("tiny", 2)
    cfg = occ_cfg(voxel_size=wl.voxel_size, num_labels=8, max_blocks=1 << 16, max_range=15.0)
    rng = np.random.default_rng(0)
    a, b = ob.OracleOcc(cfg), ob.OracleOcc(cfg)
    for pts, i in wl.scans():
        pts = pts.numpy()
        lab = rng.integers(0, 10, len(pts)).astype(np.uint16)
        conf = rng.uniform(0, 1, len(pts)).astype(np.float32)
        perm = rng.permutation(len(pts))
        a.integrate(pts, wl.pose(i), lab, conf)
        b.integrate(pts[perm], wl.pose(i), lab[perm], conf[perm])
    assert a.save_bytes() == b.save_bytes()


@needs_oracle
def test_capacity_rejects_scan_unchanged():
    o = ob.OracleOcc(occ_cfg(max_blocks=2))
    o.integrate(np.array([[0.5, 0, 0]], np.float32), svx.pose_c())
    before = o.save_bytes()
    with pytest.raises(ob.CheckerError) as e:
        o.integrate(np.array([[3.0, 0, 0]], np.float32), svx.pose_c())
    assert e.value.code == 2
    assert o.save_bytes() == before


# ------------------------------------------------------------------------ GPU

def _run_both(wl, cfg, n_frames=None, labels=True, seed=0, shard=None):
    rng = np.random.default_rng(seed)
    gpu = svx.OccupancyMap(cfg)
    if shard:
        gpu.set_shard(*shard)
    o = ob.OracleOcc(cfg)
    for pts, i in wl.scans():
        pts = pts.numpy()
        lab = rng.integers(0, cfg.num_labels + 2, len(pts)).astype(np.uint16) if labels else None
        conf = rng.uniform(-0.1, 1.1, len(pts)).astype(np.float32) if labels else None
        rg = gpu.integrate(pts, wl.pose(i), lab, conf)
        ro = o.integrate(pts, wl.pose(i), lab, conf)
        if not shard:
            assert (rg.rays, rg.hit_voxels, rg.miss_voxels, rg.new_blocks) == \
                (ro.rays, ro.hit_voxels, ro.miss_voxels, ro.new_blocks)
    return gpu, o


@pytest.mark.gpu
@needs_oracle
@pytest.mark.parametrize("variant", ["carve", "endpoints", "range_cut", "unlabelled"])
def test_gpu_occupancy_equals_oracle(variant):
    from paper_2412_00291_b200 import workload as W
    wl = W.make("tiny", 3)
    cfg = occ_cfg(voxel_size=wl.voxel_size, num_labels=20, max_blocks=1 << 17)
    if variant == "endpoints":
        cfg.carve = False
    if variant == "range_cut":
        cfg.max_range = 9.0
    gpu, o = _run_both(wl, cfg, labels=variant != "unlabelled")
    assert gpu.save_bytes() == o.save_bytes()
    # point queries agree with the export
    p = ob.parse_socc1(o.save_bytes())
    keys = p[1]
    vs = np.concatenate([keys[:50] * 8 + np.array([[1, 2, 3]]), [[10 ** 6, 0, 0]]]).astype(np.int32)
    q = gpu.lookup(vs)
    assert not q["found"][-1] and q["label"][-1] == -1
    for j in range(50):
        L, h, m, hist = voxel(p, tuple(vs[j]))
        assert q["found"][j] and q["log_odds"][j] == L and q["hits"][j] == h and q["misses"][j] == m
        if hist is not None:
            assert np.array_equal(q["hist"][j], hist)
            assert q["label"][j] == (int(np.argmax(hist)) if hist.max() > 0 else -1)
    gpu.close()


@pytest.mark.gpu
@needs_oracle
def test_gpu_occupancy_cfg2_scans_equal_oracle():
    from paper_2412_00291_b200 import workload as W
    wl = W.make("cfg2", 3)
    cfg = occ_cfg(voxel_size=wl.voxel_size, num_labels=20, max_blocks=1 << 20)
    gpu, o = _run_both(wl, cfg)
    assert gpu.save_bytes() == o.save_bytes()
    gpu.close()


def _merge_socc1(parts):
    """k-way merge of per-shard SOCC1 exports into one (sorted keys)."""
    import struct
    hdr = parts[0][:37]
    blocks = []
    for buf in parts:
        K = struct.unpack_from("<I", buf, 9)[0]
        (nb,) = struct.unpack_from("<Q", buf, 29)
        off = 37
        for _ in range(nb):
            key = tuple(np.frombuffer(buf, np.int32, 3, off))
            ln = 12 + 6144 + 1 + (2048 * K if buf[off + 12 + 6144] else 0)
            blocks.append((key, buf[off:off + ln]))
            off += ln
    blocks.sort(key=lambda kb: kb[0])
    return hdr[:29] + struct.pack("<Q", len(blocks)) + b"".join(b for _, b in blocks)


@pytest.mark.gpu
@needs_oracle
def test_gpu_occupancy_key_sharded_union_equals_unsharded():
    """two key shards (world 2) hold disjoint blocks whose union is the
    unsharded map, byte for byte."""
    from paper_2412_00291_b200 import workload as W
    wl = W.make("tiny", 2)
    cfg = occ_cfg(voxel_size=wl.voxel_size, num_labels=20, max_blocks=1 << 17)
    g0, o = _run_both(wl, cfg, shard=(0, 2))
    g1, _ = _run_both(wl, cfg, shard=(1, 2))
    assert g0.block_count() > 0 and g1.block_count() > 0
    assert _merge_socc1([g0.save_bytes(), g1.save_bytes()]) == o.save_bytes()
    g0.close()
    g1.close()


@pytest.mark.gpu
@needs_oracle
def test_gpu_occupancy_scan_completion_after_mapping(monkeypatch):
    """A scan that outruns the mapped pool is finished by a second launch that applies
    exactly the skipped updates (SVX_TEST_OCC_HEADROOM forces it on every scan)."""
    from paper_2412_00291_b200 import workload as W
    monkeypatch.setenv("SVX_TEST_OCC_HEADROOM", "3")
    wl = W.make("tiny", 3)
    cfg = occ_cfg(voxel_size=wl.voxel_size, num_labels=20, max_blocks=1 << 17)
    gpu, o = _run_both(wl, cfg)
    assert gpu.save_bytes() == o.save_bytes()
    gpu.close()


@pytest.mark.gpu
def test_gpu_occupancy_capacity_rejects_scan():
    gpu = svx.OccupancyMap(occ_cfg(max_blocks=2))
    gpu.integrate(np.array([[0.5, 0, 0]], np.float32), svx.pose_c())
    before = gpu.save_bytes()
    with pytest.raises(svx.CapacityError):
        gpu.integrate(np.array([[3.0, 0, 0]], np.float32), svx.pose_c())
    assert gpu.save_bytes() == before
    gpu.integrate(np.array([[0.5, 0, 0]], np.float32), svx.pose_c())  # still usable
    gpu.close()


# ----------------------------------------------------------- pinhole depth images
# svx.h svx_occ_integrate_depth (BASELINE.json configs[2]; no reference: unpinned).

def pinhole(w, h, f, max_depth=30.0):
    return svx.PinholeC(w, h, f, f, w / 2.0, h / 2.0, max_depth)


def back_project_np(depth, cam):
    """Independent numpy restatement of the contract's back-projection (FP64, its order)."""
    h, w = depth.shape
    v, u = np.meshgrid(np.arange(h, dtype=np.float64), np.arange(w, dtype=np.float64), indexing="ij")
    z = depth.astype(np.float64)
    keep = np.isfinite(depth) & (depth > 0) & (z <= cam.max_depth)
    with np.errstate(invalid="ignore"):
        x = ((u + 0.5 - cam.cx) * z / cam.fx).astype(np.float32)
        y = ((v + 0.5 - cam.cy) * z / cam.fy).astype(np.float32)
    pts = np.stack([x, y, depth.astype(np.float32)], -1).reshape(-1, 3)
    pts[~keep.reshape(-1)] = np.nan
    return pts


def depth_scene(n_img, w, h, seed=0):
    """Cameras on a short track looking along +x at a wall and a ground plane (z up in the
    world; camera z forward, y down), with noise, holes and far pixels."""
    rng = np.random.default_rng(seed)
    cam = pinhole(w, h, 0.8 * w, max_depth=12.0)
    # camera -> world rotation: camera z -> world +x, camera x -> world -y, camera y -> world -z
    R = np.array([[0, 0, 1], [-1, 0, 0], [0, -1, 0]], np.float64)
    imgs, poses = [], []
    for i in range(n_img):
        t = np.array([0.37 * i, 0.05 * i, 1.6])
        yaw = 0.2 * (i % 3 - 1)
        Rz = np.array([[np.cos(yaw), -np.sin(yaw), 0], [np.sin(yaw), np.cos(yaw), 0], [0, 0, 1]])
        Rw = Rz @ R
        v, u = np.meshgrid(np.arange(h) + 0.5, np.arange(w) + 0.5, indexing="ij")
        dcam = np.stack([(u - cam.cx) / cam.fx, (v - cam.cy) / cam.fy, np.ones_like(u)], -1)
        dw = dcam @ Rw.T
        t_wall = (9.0 - t[0]) / np.where(dw[..., 0] > 1e-9, dw[..., 0], np.nan)
        t_gnd = -t[2] / np.where(dw[..., 2] < -1e-9, dw[..., 2], np.nan)
        tt = np.fmin(np.where(t_wall > 0, t_wall, np.inf), np.where(t_gnd > 0, t_gnd, np.inf))
        z = (tt * 1.0).astype(np.float32)  # camera-frame z = ray parameter (dcam.z = 1)
        z += rng.normal(0, 0.01, z.shape).astype(np.float32)
        z[rng.random(z.shape) < 0.05] = 0.0       # holes
        z[rng.random(z.shape) < 0.01] = np.nan    # invalid
        z[~np.isfinite(tt)] = 0.0
        imgs.append(z.astype(np.float32))
        poses.append(svx.pose_c(Rw, t))
    labels = [rng.integers(0, 4, (h, w)).astype(np.uint16) for _ in range(n_img)]
    conf = [rng.uniform(0.2, 1.0, (h, w)).astype(np.float32) for _ in range(n_img)]
    return cam, imgs, poses, labels, conf


@needs_oracle
def test_depth_single_pixel_known_answer():
    """1x1 image, principal point at the pixel centre: depth 2 m -> point (0, 0, 2): one
    HIT at voxel (0, 0, 20), MISS for the 20 cells from the camera to it."""
    o = ob.OracleOcc(occ_cfg())
    cam = svx.PinholeC(1, 1, 100.0, 100.0, 0.5, 0.5, 30.0)
    r = o.integrate_depth(np.array([[2.0]], np.float32), cam, svx.pose_c())
    assert (r.points, r.rays, r.hit_voxels, r.miss_voxels) == (1, 1, 1, 20)
    p = ob.parse_socc1(o.save_bytes())
    assert voxel(p, (0, 0, 20))[:3] == (np.float32(0.85), 1, 0)
    assert voxel(p, (0, 0, 7))[:3] == (np.float32(-0.4), 0, 1)


@needs_oracle
def test_depth_dropped_pixels():
    """0, negative, NaN, inf and beyond-max_depth pixels are not rays."""
    o = ob.OracleOcc(occ_cfg())
    cam = svx.PinholeC(6, 1, 10.0, 10.0, 3.0, 0.5, 5.0)
    d = np.array([[0.0, -1.0, np.nan, np.inf, 5.5, 5.0]], np.float32)
    r = o.integrate_depth(d, cam, svx.pose_c())
    assert (r.points, r.rays, r.hit_voxels) == (6, 1, 1)


@needs_oracle
def test_depth_equals_point_cloud_path():
    """The oracle's depth path == its point path on an independently back-projected
    cloud (numpy restatement of the contract's arithmetic)."""
    cam, imgs, poses, labels, conf = depth_scene(3, 40, 30)
    a, b = ob.OracleOcc(occ_cfg(max_blocks=1 << 14)), ob.OracleOcc(occ_cfg(max_blocks=1 << 14))
    for d, p, lb, cf in zip(imgs, poses, labels, conf):
        ra = a.integrate_depth(d, cam, p, lb, cf)
        rb = b.integrate(back_project_np(d, cam), p, lb.reshape(-1), cf.reshape(-1))
        assert (ra.rays, ra.hit_voxels, ra.miss_voxels) == (rb.rays, rb.hit_voxels, rb.miss_voxels)
        assert ra.rays > 0.8 * d.size
    assert a.save_bytes() == b.save_bytes()


def test_depth_api_rejects_bad_arguments():
    m = svx.OccupancyMap.__new__(svx.OccupancyMap)  # argument checks happen before any GPU call
    cam = pinhole(4, 3, 3.0)
    with pytest.raises(svx.InvalidArgument):
        svx.OccupancyMap.integrate_depth(m, [np.zeros((4, 4), np.float32)], [cam], [svx.pose_c()])
    with pytest.raises(svx.InvalidArgument):
        svx.OccupancyMap.integrate_depth(m, [np.zeros((3, 4), np.float32)], [cam], [])


@pytest.mark.gpu
@needs_oracle
def test_gpu_depth_images_equal_oracle():
    """Two 'frames' of 3 labelled depth cameras: GPU SOCC1 == oracle SOCC1, host and
    device-pointer entry points agree."""
    import torch
    cam, imgs, poses, labels, conf = depth_scene(6, 96, 64, seed=3)
    cfg = occ_cfg(max_blocks=1 << 15)
    o = ob.OracleOcc(cfg)
    g = svx.OccupancyMap(cfg, 0)
    g2 = svx.OccupancyMap(cfg, 0)
    for f in (0, 3):
        sl = slice(f, f + 3)
        rg = g.integrate_depth(imgs[sl], [cam] * 3, poses[sl], labels[sl], conf[sl])
        dd = torch.from_numpy(np.concatenate([x.reshape(-1) for x in imgs[sl]])).cuda()
        dl = torch.from_numpy(np.concatenate([x.reshape(-1) for x in labels[sl]]).view(np.int16)).cuda()
        dc = torch.from_numpy(np.concatenate([x.reshape(-1) for x in conf[sl]])).cuda()
        torch.cuda.synchronize()
        r2 = g2.integrate_depth_device(dd.data_ptr(), [cam] * 3, poses[sl], dl.data_ptr(), dc.data_ptr())
        for j in range(3):
            ro = o.integrate_depth(imgs[f + j], cam, poses[f + j], labels[f + j], conf[f + j])
            assert (rg[j].rays, rg[j].hit_voxels, rg[j].miss_voxels, rg[j].new_blocks) == \
                (ro.rays, ro.hit_voxels, ro.miss_voxels, ro.new_blocks)
            assert (r2[j].hit_voxels, r2[j].miss_voxels) == (ro.hit_voxels, ro.miss_voxels)
    ref = o.save_bytes()
    assert g.save_bytes() == ref
    assert g2.save_bytes() == ref
    g.close()
    g2.close()


# ------------------------------------------------------- C++ host API (drop-in)
DROPIN_TEST = svx.LIB_PATH.replace("libsvx_b200.so", "test_occupancy_dropin")


def test_cpp_occupancy_api_is_built():
    """semvox/occupancy_map.hpp is compiled into libsemvox_b200.so and its check
    program is built in-tree (make -C paper_2412_00291_b200/csrc)."""
    import os
    assert os.access(DROPIN_TEST, os.X_OK), DROPIN_TEST
    import ctypes
    lib = ctypes.CDLL(svx.LIB_PATH.replace("libsvx_b200.so", "libsemvox_b200.so"))
    assert hasattr(lib, "_ZN6semvox12OccupancyMap15integrate_depthERKSt6vectorINS_10DepthImageESaIS2_EE")


@pytest.mark.gpu
def test_gpu_cpp_occupancy_api():
    """The C++ OccupancyMap reproduces the contract's known answers on the device."""
    import subprocess
    r = subprocess.run([DROPIN_TEST], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all checks passed" in r.stdout
