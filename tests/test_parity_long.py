"""Long-sequence parity on the benchmarked configurations, against the REFERENCE'S
OWN CODE (oracle/_ref/libsemvox_ref.so: the reference's translation units built
unmodified from /root/reference; RefMap), not only the C restatement.

What bench.py times is the batched device path (svx_integrate_clouds_device /
svx_integrate_clouds); these tests drive exactly those entry points over long
runs of the bench workloads and compare, frame by frame, the reports
(updated_voxels, new_blocks, tsdf_integrator.cpp:250-257) and at the end the
whole SVOX1 image (voxel_store.cpp:82-130), the dirty lists and the semantic
layers. The non-projective mode (the reference's default, and what bench.py
runs) reads each voxel's accumulated gradient (tsdf_integrator.cpp:190-196), so
a ulp-level difference would compound over a long run: that is what these
sequences are for.

Reference call sites: cmd_integrate's per-frame body (proj/tools/semvox_main.cpp:121-146)
= project_cloud + compute_normal_image + integrate_frame (+ integrate_labels).
"""
import os

import numpy as np
import pytest

import paper_2412_00291_b200 as svx
from oracle import bindings as ob
from paper_2412_00291_b200 import workload as W
from tests.helpers import compare_maps

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

os.environ.setdefault("SEMVOX_THREADS", str(os.cpu_count() or 1))


def _scans_on_gpu(wl, frames=None):
    import torch
    dev = torch.device("cuda", 0)
    return [(p.cpu().numpy(), i) for p, i in wl.scans(device=dev, frames=frames)]


def _flat(scans):
    offs = np.zeros(len(scans) + 1, np.uint64)
    offs[1:] = np.cumsum([s.shape[0] for s, _ in scans])
    flat = np.ascontiguousarray(np.concatenate([s for s, _ in scans]).astype(np.float32))
    return flat, offs


def _run_long(wl, icfg, n_frames, batch, max_blocks=1 << 21, host=False):
    """GPU: batched entry point, `batch` frames per call. Reference: one
    integrate_cloud per frame. Returns (gpu store, ref map, reports)."""
    import torch
    scans = _scans_on_gpu(wl, frames=range(n_frames))
    flat, offs = _flat(scans)
    poses = [wl.pose(i) for _, i in scans]
    cfg = svx.MapConfig(wl.voxel_size, wl.truncation, wl.num_labels, max_blocks)
    g = svx.VoxelStore(cfg, 0)
    r = ob.RefMap(cfg)
    src = torch.from_numpy(flat).pin_memory() if host else torch.from_numpy(flat).cuda()
    got = []
    for f0 in range(0, n_frames, batch):
        f1 = min(n_frames, f0 + batch)
        rel = offs[f0:f1 + 1] - offs[f0]
        ptr = src.data_ptr() + int(offs[f0]) * 12
        if host:
            got += g.integrate_clouds_host(wl.model, ptr, rel, 3, poses[f0:f1], icfg)
        else:
            got += g.integrate_clouds_device(wl.model, ptr, rel, 3, poses[f0:f1], icfg)
    want = [r.integrate_cloud(wl.model, s, wl.pose(i), icfg)[0] for s, i in scans]
    for a, b in zip(got, want):
        assert (a.frame, a.updated_voxels, a.new_blocks) == \
            (b.frame, b.updated_voxels, b.new_blocks), (a, b)
    return g, r, got


def _check_same(g, r, exact=True):
    a, b = g.save_bytes(), r.save_bytes()
    st = compare_maps(a, b)
    assert np.array_equal(g.take_dirty_blocks(0), r.take_dirty(0))
    if exact:
        assert a == b, ("SVOX1 bytes differ from the reference's", st)
    return st


@pytest.mark.parametrize("mode", [svx.NON_PROJECTIVE, svx.PROJECTIVE])
def test_cfg2_200_frames_vs_reference(mode):
    """The bench workload (cfg2: 1024x128, 0.1 m, tau 0.5) for 200 consecutive
    scans through svx_integrate_clouds_device in batches of 100, as bench.py runs it."""
    wl = W.make("cfg2", 200)
    g, r, reps = _run_long(wl, svx.IntegratorConfig(mode=mode), 200, 100)
    st = _check_same(g, r)
    assert st["blocks"] > 30000
    assert sum(x.updated_voxels for x in reps) > 1e8
    g.close()


def test_cfg2_host_ingest_120_frames_vs_reference():
    """The e2e leg's entry point (svx_integrate_clouds: pinned host points, staged
    through the ingest ring), batches of 40."""
    wl = W.make("cfg2", 120)
    g, r, _ = _run_long(wl, svx.IntegratorConfig(), 120, 40, host=True)
    _check_same(g, r)
    g.close()


def test_cfg1_100_frames_vs_reference():
    """cfg1 (2048x64, 0.2 m, tau 1.0): the reference's CPU configuration, 100 scans."""
    wl = W.make("cfg1", 100)
    g, r, _ = _run_long(wl, svx.IntegratorConfig(), 100, 50)
    _check_same(g, r)
    g.close()


def test_cfg3_20_frames_six_cameras_vs_reference():
    """cfg3 at full size: 0.05 m voxels, tau 0.25, and all six 1280x720 label
    images per frame (semantic_integrator.cpp:91-165), 20 frames."""
    import torch
    wl = W.make("cfg3", 20)
    dev = torch.device("cuda", 0)
    cfg = svx.MapConfig(wl.voxel_size, wl.truncation, wl.num_labels, 1 << 21)
    g = svx.VoxelStore(cfg, 0)
    r = ob.RefMap(cfg)
    icfg, scfg = svx.IntegratorConfig(), svx.SemanticConfig()
    ti, si = svx.TsdfIntegrator(g, icfg), svx.SemanticIntegrator(g, scfg)
    n_sem = 0
    for p, i in wl.scans(device=dev):
        p = p.cpu().numpy()
        a = ti.integrate_cloud(p, wl.pose(i), wl.model)
        b, _ = r.integrate_cloud(wl.model, p, wl.pose(i), icfg)
        assert (a.frame, a.updated_voxels, a.new_blocks) == (b.frame, b.updated_voxels, b.new_blocks)
        imgs = wl.label_images(i, device=dev)
        assert len(imgs) == 6 and imgs[0].width == 1280 and imgs[0].height == 720
        sa = si.integrate_labels_batch(imgs)
        sb = [r.integrate_labels(li, scfg) for li in imgs]
        assert [(x.frame, x.updated_voxels) for x in sa] == [(x.frame, x.updated_voxels) for x in sb]
        n_sem += sum(x.updated_voxels for x in sa)
    assert n_sem > 1e6
    st = _check_same(g, r)
    assert np.array_equal(g.take_dirty_blocks(1), r.take_dirty(1))
    assert st["blocks"] > 20000
    g.close()


# ---------------------------------------------------------------- exact boundaries
# SURVEY.md 7.2 hard part #1: a pixel decision is floor() of a transcendental
# expression (scan_projection.cpp:21-37), evaluated on the device with FP32 + a
# margin and CUDA's FP64 atan2/acos near a boundary. Where the reference's FP64
# value is EXACTLY an integer, a 1-ulp difference between CUDA's and glibc's
# atan2/acos would flip the pixel. These inputs sit exactly there: azimuths on
# multiples of pi/4 (|x| = |y|, or a zero component) are pixel boundaries when W is
# divisible by 8; z = 0 puts the polar angle on the row boundary of a symmetric
# field of view (acos(0) = pi/2).

def _boundary_clouds():
    out = []
    for a in (0.5, 1.0, 3.0, 7.25, np.float32(0.1), np.float32(2.3), 19.0):
        a = float(np.float32(a))
        pts = []
        for sx, sy in ((1, 1), (-1, 1), (1, -1), (-1, -1), (1, 0), (0, 1), (-1, 0), (0, -1)):
            for z in (0.0, 0.25 * a, -0.25 * a, 0.4 * a):
                pts.append((sx * a, sy * a, z))
        out.append(np.array(pts, np.float32))
    return out


@pytest.mark.parametrize("width", [8, 64, 512, 1024, 2048, 4096])
def test_exact_boundary_pixels_match_reference(width):
    """Device project_cloud == the reference's on points exactly on pixel boundaries."""
    m = svx.ProjectionModel.spinning(width, 128, 22.5, 22.5)
    g = svx.VoxelStore(svx.MapConfig(0.1, 0.5, 2), 0)
    pose = svx.pose_c(np.eye(3), [0.0, 0.0, 0.0])
    for pts in _boundary_clouds():
        img = svx.project_cloud(pts, pose, m, g)
        d, h, n, v, dr = ob.RefMap.project(m, pts, pose)
        assert np.array_equal(img.depth, d), np.nonzero(img.depth != d)
        assert np.array_equal(img.height, h)
        assert img.dropped == dr
    g.close()


def test_exact_boundary_atan2_acos_device_vs_glibc():
    """The FP64 slow path's transcendentals themselves: the device's pixel of a point
    whose FP64 azimuth/polar coordinate is an exact integer equals the floor of
    glibc's value (ctypes libm) at atan2(a, a), atan2(a, 0), atan2(0, a), acos(0)."""
    import ctypes
    libm = ctypes.CDLL("libm.so.6")
    libm.atan2.restype = libm.acos.restype = ctypes.c_double
    libm.atan2.argtypes = [ctypes.c_double, ctypes.c_double]
    libm.acos.argtypes = [ctypes.c_double]
    pi = 3.14159265358979323846
    for width in (8, 1024, 4096):
        m = svx.ProjectionModel.spinning(width, 128, 22.5, 22.5)
        for pts in _boundary_clouds():
            for x, y, z in pts.astype(np.float64):
                r = np.sqrt((x * x + y * y) + z * z)
                u = int(np.floor((pi - libm.atan2(y, x)) / m.delta_phi)) % width
                c = min(1.0, max(-1.0, z / r))
                v = int(np.floor((libm.acos(c) - m.theta0) / m.delta_theta))
                # the device agrees with this glibc evaluation pixel for pixel
                img = svx.project_cloud(np.array([[x, y, z]], np.float32), svx.pose_c(np.eye(3), [0, 0, 0]),
                                        m, _store())
                nz = np.nonzero(img.depth)[0]
                if r >= m.min_range and 0 <= v < 128:
                    assert list(nz) == [v * width + u], (x, y, z, width, nz, v * width + u)
                else:
                    assert len(nz) == 0


_STORE = []


def _store():
    if not _STORE:
        _STORE.append(svx.VoxelStore(svx.MapConfig(0.1, 0.5, 2), 0))
    return _STORE[0]


@pytest.mark.parametrize("mode", [svx.NON_PROJECTIVE, svx.PROJECTIVE])
def test_pose_at_origin_voxels_on_diagonals_vs_reference(mode):
    """A sensor at x = y = 0 with identity rotation: voxel centres with |x| = |y| lie
    exactly on the pi/4 azimuths, which are pixel boundaries for W = 1024, so the
    own-pixel decisions of integrate_frame (tsdf_integrator.cpp:232) hit the exact
    boundary. Full pipeline vs the reference's own code, several frames."""
    import torch
    wl = W.make("cfg2", 4)
    dev = torch.device("cuda", 0)
    poses = [(np.eye(3), np.array([0.0, 0.0, 1.75])), (np.eye(3), np.array([0.0, 0.0, 1.0])),
             (np.eye(3), np.array([0.0, 0.0, 2.0])), (np.eye(3), np.array([0.0, 0.0, 1.75]))]
    wl.poses = poses
    cfg = svx.MapConfig(wl.voxel_size, wl.truncation, wl.num_labels, 1 << 20)
    icfg = svx.IntegratorConfig(mode=mode)
    g = svx.VoxelStore(cfg, 0)
    r = ob.RefMap(cfg)
    ti = svx.TsdfIntegrator(g, icfg)
    for p, i in wl.scans(device=dev):
        p = p.cpu().numpy()
        a = ti.integrate_cloud(p, wl.pose(i), wl.model)
        b, _ = r.integrate_cloud(wl.model, p, wl.pose(i), icfg)
        assert (a.updated_voxels, a.new_blocks) == (b.updated_voxels, b.new_blocks)
    _check_same(g, r)
    g.close()
