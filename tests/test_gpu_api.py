"""GPU: the reference's own unit-test scenarios (proj/tests/test_voxel_store.cpp,
test_scan_projection.cpp, test_tsdf_integrator.cpp, test_semantic_integrator.cpp)
restated against the B200 library through the C-ABI."""
import math
import os

import numpy as np
import pytest

import paper_2412_00291_b200 as svx
from paper_2412_00291_b200 import TSDF_DTYPE

pytestmark = pytest.mark.gpu


def vc_block(v):
    return tuple(int(np.floor_divide(x, 8)) for x in v)


# ------------------------------------------------------------- voxel store

def test_allocation_idempotent_and_unobserved():        # test_voxel_store.cpp:36-51
    s = svx.VoxelStore(svx.MapConfig(num_labels=4))
    assert s.get_or_allocate_block((0, 0, 0)) is True
    assert s.get_or_allocate_block((0, 0, 0)) is False
    assert s.block_count() == 1
    s.get_or_allocate_block((1, 0, 0))
    assert s.block_count() == 2
    t, p = s.lookup_voxel((3, 3, 3))
    assert t["weight"] == 0.0 and np.allclose(p, 0.25)


def test_capacity_budget():                              # :53-62
    s = svx.VoxelStore(svx.MapConfig(max_blocks=2))
    s.get_or_allocate_block((0, 0, 0))
    s.get_or_allocate_block((1, 0, 0))
    with pytest.raises(svx.CapacityError):
        s.get_or_allocate_block((2, 0, 0))
    s.get_or_allocate_block((0, 0, 0))


def test_lookup_never_allocates_negative_coords():       # :64-75
    s = svx.VoxelStore(svx.MapConfig())
    assert s.lookup_voxel((5, 5, 5)) is None and s.block_count() == 0
    s.get_or_allocate_block((-1, -1, -1))
    assert s.lookup_voxel((-1, -1, -1)) is not None
    assert s.lookup_voxel((0, 0, 0)) is None
    t = np.zeros(512, TSDF_DTYPE)
    t["weight"][7 + 8 * 7 + 64 * 7] = 2.5                 # local_index(-1,-1,-1) = 511
    s.write_block((-1, -1, -1), t)
    assert s.lookup_voxel((-1, -1, -1))[0]["weight"] == 2.5


def test_stats_counts():                                  # :77-92
    s = svx.VoxelStore(svx.MapConfig())
    assert s.stats().allocated_blocks == 0 and s.stats().observed_voxels == 0
    s.get_or_allocate_block((0, 0, 0))
    st = s.stats()
    assert st.allocated_blocks == 1 and st.observed_voxels == 0 and st.memory_bytes > 0
    t = np.zeros(512, TSDF_DTYPE)
    t["weight"][0], t["weight"][100] = 1.0, 0.5
    s.write_block((0, 0, 0), t)
    assert s.stats().observed_voxels == 2


def test_dense_residency_32cubed():                       # :94-124
    s = svx.VoxelStore(svx.MapConfig(voxel_size=0.1, truncation=0.5))
    n = 32
    rng = np.random.default_rng(11)
    dense = rng.uniform(-0.5, 0.5, (n, n, n)).astype(np.float32)
    blocks = {}
    for z in range(n):
        for y in range(n):
            for x in range(n):
                v = (x - n // 2, y - n // 2, z - n // 2)
                b = vc_block(v)
                if b not in blocks:
                    blocks[b] = np.zeros(512, TSDF_DTYPE)
                li = (v[0] % 8) + 8 * (v[1] % 8) + 64 * (v[2] % 8)
                blocks[b]["distance"][li] = dense[z, y, x]
                blocks[b]["weight"][li] = 1.0
    for b, t in blocks.items():
        s.write_block(b, t)
    zz, yy, xx = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    coords = np.stack([xx - n // 2, yy - n // 2, zz - n // 2], -1).reshape(-1, 3)
    f, t, _ = s.lookup_voxels(coords)
    assert f.all()
    assert np.array_equal(t["distance"], dense.reshape(-1))


def test_snapshot_round_trip_bit_exact(tmp_path):         # :138-182
    cfg = svx.MapConfig(0.25, 1.25, 3)
    s = svx.VoxelStore(cfg)
    rng = np.random.default_rng(23)
    for bc in ((0, 0, 0), (-2, 1, 5), (7, -3, 0)):
        t = np.zeros(512, TSDF_DTYPE)
        t["distance"] = rng.uniform(-1, 1, 512)
        t["weight"] = np.abs(rng.uniform(-1, 1, 512))
        g = rng.uniform(-1, 1, (512, 3)).astype(np.float32)
        t["gradient"] = g / np.linalg.norm(g, axis=1, keepdims=True)
        s.write_block(bc, t)
    sem = np.full((512, 3), np.float32(1.0) / np.float32(3.0), np.float32)
    sem[0] = [0.8, 0.15, 0.05]
    s.write_block((0, 0, 0), s.read_block((0, 0, 0))[0], sem)
    p1, p2 = tmp_path / "a.svox", tmp_path / "b.svox"
    s.save(str(p1))
    loaded = svx.VoxelStore.load(str(p1))
    loaded.save(str(p2))
    assert p1.read_bytes() == p2.read_bytes()
    assert loaded.config().num_labels == 3 and loaded.block_count() == 3
    assert loaded.lookup_voxel((0, 0, 0))[1][0] == np.float32(0.8)
    assert loaded.read_block((-2, 1, 5))[1] is None       # lazy layer preserved
    with pytest.raises(svx.DataError):
        svx.VoxelStore.load(str(tmp_path / "missing.svox"))


def test_load_rejects_garbage_and_caps_blocks(tmp_path):
    p = tmp_path / "x.svox"
    p.write_bytes(b"NOTSVOX")
    with pytest.raises(svx.DataError):
        svx.VoxelStore.load(str(p))
    s = svx.VoxelStore(svx.MapConfig())
    for i in range(5):
        s.get_or_allocate_block((i, 0, 0))
    s.save(str(p))
    with pytest.raises(svx.CapacityError):
        svx.VoxelStore.load(str(p), max_blocks=4)


def test_block_keys_sorted():
    s = svx.VoxelStore(svx.MapConfig())
    keys = [(3, 1, 1), (-1, 5, 0), (3, 0, 9), (-1, 5, -2)]
    for k in keys:
        s.get_or_allocate_block(k)
    assert [tuple(k) for k in s.block_coords_sorted()] == sorted(keys)


# ------------------------------------------------------------- projection

def plane_scan(model, sensor, plane_z):
    """test_tsdf_integrator.cpp:19-31"""
    from paper_2412_00291_b200.workload import pixel_dirs
    d = pixel_dirs(model).numpy()
    ok = d[:, 2] < -1e-3
    t = (plane_z - sensor[2]) / d[ok, 2]
    keep = (t >= model.min_range) & (t <= 50.0)
    return (d[ok][keep] * t[keep, None]).astype(np.float32), svx.pose_c(np.eye(3), sensor)


def test_plane_normals_vertical():                        # test_scan_projection.cpp:113-138
    m = svx.ProjectionModel.spinning(1024, 64, 22.5, 22.5)
    s = svx.VoxelStore(svx.MapConfig())
    pts, pose = plane_scan(m, (0, 0, 2.0), 0.0)
    img = svx.project_cloud(pts, pose, m, s)
    n = img.normals[img.normal_valid.astype(bool)]
    assert len(n) > 1000
    assert np.allclose(np.linalg.norm(n, axis=1), 1.0, atol=1e-5)
    assert np.all(n[:, 2] > 0) and np.allclose(np.abs(n[:, 2]), 1.0, atol=1e-3)


def test_degenerate_neighbours_no_normal():               # :140-155
    m = svx.ProjectionModel.spinning(16, 8, 30, 30)
    s = svx.VoxelStore(svx.MapConfig())
    d = np.zeros(128, np.float32)
    d[5 * 16 + 5] = 2.0
    img = svx.compute_normal_image(svx.ScanImages(m, d, np.zeros(128, np.float32)), s)
    assert img.normal_valid[5 * 16 + 5] == 0
    img = svx.compute_normal_image(svx.ScanImages(m, np.ones(128, np.float32),
                                                  np.zeros(128, np.float32)), s)
    assert not img.normal_valid[:16].any()


def test_bad_pose_rejected():
    m = svx.ProjectionModel.spinning(64, 8, 20, 20)
    s = svx.VoxelStore(svx.MapConfig())
    with pytest.raises(svx.InvalidArgument):
        svx.project_cloud(np.ones((4, 3), np.float32), svx.pose_c(np.eye(3) * 2.0), m, s)


# ------------------------------------------------------------- TSDF

def test_single_ray_band():                               # test_tsdf_integrator.cpp:166-207
    s = svx.VoxelStore(svx.MapConfig(0.1, 0.5))
    ti = svx.TsdfIntegrator(s, svx.IntegratorConfig(mode=svx.PROJECTIVE))
    m = svx.ProjectionModel.spinning(1024, 64, 22.5, 22.5)
    r = ti.integrate_cloud(np.array([[2.0, 0, 0]], np.float32), svx.pose_c(), m)
    assert r.updated_voxels >= 8 and r.new_blocks > 0
    hit = s.lookup_voxel((20, 0, 0))
    assert hit is not None and abs(float(hit[0]["distance"])) <= 0.1


def test_empty_depth_image():                             # :209-223
    s = svx.VoxelStore(svx.MapConfig())
    m = svx.ProjectionModel.spinning(64, 16, 20, 20)
    img = svx.ScanImages(m, np.zeros(1024, np.float32), np.zeros(1024, np.float32),
                         np.zeros((1024, 3), np.float32), np.zeros(1024, np.uint8))
    r = svx.TsdfIntegrator(s).integrate_frame(img, svx.pose_c())
    assert (r.updated_voxels, r.new_blocks, s.block_count()) == (0, 0, 0)


def test_nonprojective_needs_normals():                   # tsdf_integrator.cpp:102-103
    s = svx.VoxelStore(svx.MapConfig())
    m = svx.ProjectionModel.spinning(64, 16, 20, 20)
    img = svx.ScanImages(m, np.ones(1024, np.float32), np.zeros(1024, np.float32))
    with pytest.raises(svx.InvalidArgument):
        svx.TsdfIntegrator(s).integrate_frame(img, svx.pose_c())
    with pytest.raises(svx.InvalidArgument):
        svx.TsdfIntegrator(s, svx.IntegratorConfig(alpha_epsilon=0.0))


def test_repeated_frames_fixed_point():                   # :225-250
    s = svx.VoxelStore(svx.MapConfig(0.1, 0.5))
    m = svx.ProjectionModel.spinning(256, 32, 25, 25)
    pts, pose = plane_scan(m, (0, 0, 1.5), 0.0)
    ti = svx.TsdfIntegrator(s)
    ti.integrate_cloud(pts, pose, m)
    a = s.save_bytes()
    ti.integrate_cloud(pts, pose, m)
    from oracle.bindings import parse_svox1
    _, ka, ta, _ = parse_svox1(a)
    _, kb, tb, _ = parse_svox1(s.save_bytes())
    obs = ta["weight"] > 0
    assert np.array_equal(ka, kb)
    assert np.allclose(tb["distance"][obs], ta["distance"][obs], atol=1e-5)
    assert np.allclose(tb["weight"][obs], 2 * ta["weight"][obs], rtol=1e-5)


def test_band_and_unit_gradients():                       # :252-274
    s = svx.VoxelStore(svx.MapConfig(0.1, 0.3))
    m = svx.ProjectionModel.spinning(256, 32, 25, 25)
    ti = svx.TsdfIntegrator(s)
    for i in range(5):
        pts, pose = plane_scan(m, (0.3 * i, 0, 1.0 + 0.2 * i), 0.0)
        ti.integrate_cloud(pts, pose, m)
    from oracle.bindings import parse_svox1
    _, _, t, _ = parse_svox1(s.save_bytes())
    obs = t["weight"] > 0
    assert obs.sum() > 1000
    assert np.all(np.abs(t["distance"][obs]) <= 0.3 + 1e-6)
    gn = np.linalg.norm(t["gradient"][obs], axis=1)
    assert np.all((np.abs(gn - 1) < 1e-5) | (gn == 0))


def test_permuted_input_identical_map():                  # :276-298
    m = svx.ProjectionModel.spinning(256, 32, 25, 25)
    pts, pose = plane_scan(m, (0, 0, 1.5), 0.0)
    maps = []
    for perm in (np.arange(len(pts)), np.random.default_rng(9).permutation(len(pts))):
        s = svx.VoxelStore(svx.MapConfig(0.1, 0.5))
        svx.TsdfIntegrator(s).integrate_cloud(pts[perm], pose, m)
        maps.append(s.save_bytes())
    assert maps[0] == maps[1]


def test_weights_monotone():                              # :381-403
    s = svx.VoxelStore(svx.MapConfig(0.1, 0.5))
    m = svx.ProjectionModel.spinning(128, 32, 30, 30)
    ti = svx.TsdfIntegrator(s)
    from oracle.bindings import parse_svox1
    last = {}
    for i in range(4):
        pts, pose = plane_scan(m, (0.2 * i, 0, 1.2), 0.0)
        ti.integrate_cloud(pts, pose, m)
        _, k, t, _ = parse_svox1(s.save_bytes())
        for j, kk in enumerate(map(tuple, k)):
            if kk in last:
                assert np.all(t["weight"][j] >= last[kk])
            last[kk] = t["weight"][j].copy()


# ------------------------------------------------------------- semantics

def store_with_voxel(cfg, world, distance=0.0):         # test_semantic_integrator.cpp:12-19
    s = svx.VoxelStore(cfg)
    inv = 1.0 / float(np.float32(cfg.voxel_size))
    vc = tuple(int(math.floor(c * inv + 0.5)) for c in world)
    t = np.zeros(512, TSDF_DTYPE)
    li = (vc[0] % 8) + 8 * (vc[1] % 8) + 64 * (vc[2] % 8)
    t["weight"][li], t["distance"][li] = 1.0, distance
    s.write_block(vc_block(vc), t)
    return s, vc


def simple_image(label, K=2):
    return svx.LabelImage(8, 8, np.full(64, label, np.uint16), 8.0, 8.0, 4.0, 4.0, svx.pose_c())


def test_semantic_skips():                                # :101-131
    cfg = svx.MapConfig(0.25, 1.25, 2)
    s, _ = store_with_voxel(cfg, (0, 0, -2.0))
    assert svx.SemanticIntegrator(s).integrate_labels(simple_image(0)).updated_voxels == 0
    s = svx.VoxelStore(cfg)
    s.get_or_allocate_block((0, 0, 1))
    assert svx.SemanticIntegrator(s).integrate_labels(simple_image(0)).updated_voxels == 0
    s, _ = store_with_voxel(cfg, (0, 0, 2.0))
    img = simple_image(0)
    img.max_depth = 1.0
    assert svx.SemanticIntegrator(s).integrate_labels(img).updated_voxels == 0
    s, _ = store_with_voxel(cfg, (0, 0, 2.0), -0.7)
    assert svx.SemanticIntegrator(s).integrate_labels(simple_image(0)).updated_voxels == 0


def test_semantic_tensor_stored():                        # :133-151
    cfg = svx.MapConfig(0.25, 1.25, 2)
    s, vc = store_with_voxel(cfg, (0, 0, 2.0))
    img = simple_image(0)
    img.prob_tensor = np.tile(np.array([0.7, 0.3], np.float32), (64, 1))
    assert svx.SemanticIntegrator(s).integrate_labels(img).updated_voxels == 1
    p = s.lookup_voxel(vc)[1]
    assert p[0] == pytest.approx(0.7, rel=1e-5) and p[1] == pytest.approx(0.3, rel=1e-5)


def test_no_bayes_latest_argmax():                        # :202-218
    cfg = svx.MapConfig(0.25, 1.25, 3)
    s, vc = store_with_voxel(cfg, (0, 0, 2.0))
    si = svx.SemanticIntegrator(s, svx.SemanticConfig(use_bayes=False))
    si.integrate_labels(simple_image(1))
    si.integrate_labels(simple_image(2))
    p = s.lookup_voxel(vc)[1]
    assert int(np.argmax(p)) == 2 and p[2] == 1.0 and p[1] == 0.0


def test_lazy_semantic_layers():                          # :220-231
    cfg = svx.MapConfig(0.25, 1.25, 2)
    s, vc = store_with_voxel(cfg, (0, 0, 2.0))
    s.get_or_allocate_block((100, 0, 0))
    svx.SemanticIntegrator(s).integrate_labels(simple_image(0))
    assert s.read_block(vc_block(vc))[1] is not None
    assert s.read_block((100, 0, 0))[1] is None
    dirty = s.take_dirty_blocks(1)
    assert [tuple(d) for d in dirty] == [vc_block(vc)]


def test_raycast_occlusion():                             # :233-276
    cfg = svx.MapConfig(0.1, 0.5, 2)
    s = svx.VoxelStore(cfg)
    blocks = {}
    for zi in range(8, 13):
        for dy in range(-3, 4):
            for dx in range(-3, 4):
                b = vc_block((dx, dy, zi))
                blocks.setdefault(b, np.zeros(512, TSDF_DTYPE))
                li = (dx % 8) + 8 * (dy % 8) + 64 * (zi % 8)
                blocks[b]["weight"][li] = 1.0
                blocks[b]["distance"][li] = np.float32(1.0 - 0.1 * zi)
    target = (0, 0, 20)
    b = vc_block(target)
    blocks.setdefault(b, np.zeros(512, TSDF_DTYPE))
    blocks[b]["weight"][(0) + 64 * (20 % 8)] = 1.0
    for k, t in blocks.items():
        s.write_block(k, t)
    img = simple_image(0)
    img.max_depth = 10.0
    svx.SemanticIntegrator(s, svx.SemanticConfig(occlusion=svx.RAYCAST)).integrate_labels(img)
    assert s.lookup_voxel(target)[1][0] == pytest.approx(0.5)
    assert s.lookup_voxel((0, 0, 10))[1][0] > 0.5


def test_invalid_confidence_rejected():
    cfg = svx.MapConfig(0.25, 1.25, 2)
    s, _ = store_with_voxel(cfg, (0, 0, 2.0))
    img = simple_image(0)
    img.confidence = np.full(64, 1.5, np.float32)
    with pytest.raises(svx.InvalidArgument):
        svx.SemanticIntegrator(s).integrate_labels(img)


def test_invalid_confidence_only_where_read():
    """label_to_likelihood throws only for a pixel that a voxel passing every test
    reads (semantic_integrator.cpp:24-27,140-142): an invalid confidence elsewhere,
    or an invalid default on a frame no voxel passes, integrates normally."""
    cfg = svx.MapConfig(0.25, 1.25, 2)
    s, vc = store_with_voxel(cfg, (0, 0, 2.0))
    si = svx.SemanticIntegrator(s)
    img = simple_image(0)
    img.confidence = np.full(64, 0.8, np.float32)
    img.confidence[0] = 7.0                  # no voxel projects to pixel (0, 0)
    r = si.integrate_labels(img)
    assert r.updated_voxels == 1 and r.frame == 0
    assert s.lookup_voxel(vc)[1][0] == pytest.approx(0.8)
    img.confidence[4 * 8 + 4] = -0.5         # the voxel's own pixel: throws, updates nothing
    before = s.save_bytes()
    with pytest.raises(svx.InvalidArgument):
        si.integrate_labels(img)
    assert s.save_bytes() == before
    img.confidence[4 * 8 + 4] = np.nan       # NaN passes the reference's comparison
    assert si.integrate_labels(img).frame == 2
    # invalid default confidence: fine while no voxel passes, throws once one does
    bad = svx.SemanticIntegrator(svx.VoxelStore(cfg), svx.SemanticConfig(default_confidence=1.5))
    assert bad.integrate_labels(simple_image(0)).updated_voxels == 0
    s2, _ = store_with_voxel(cfg, (0, 0, 2.0))
    with pytest.raises(svx.InvalidArgument):
        svx.SemanticIntegrator(s2, svx.SemanticConfig(default_confidence=1.5)).integrate_labels(
            simple_image(0))


def test_invalid_confidence_batch_stops_at_failing_image():
    cfg = svx.MapConfig(0.25, 1.25, 2)
    s, vc = store_with_voxel(cfg, (0, 0, 2.0))
    imgs = [simple_image(0), simple_image(1), simple_image(0)]
    for im in imgs:
        im.confidence = np.full(64, 0.7, np.float32)
    imgs[1].confidence[36] = 2.0
    si = svx.SemanticIntegrator(s)
    with pytest.raises(svx.InvalidArgument):
        si.integrate_labels_batch(imgs)
    # only image 0 was applied; images 0 and 1 are numbered
    assert s.lookup_voxel(vc)[1][0] == pytest.approx(0.7)
    assert si.integrate_labels(simple_image(0)).frame == 2


def test_key_range_abort_leaves_no_partial_blocks():
    """A frame whose band leaves the device key range [-2^20, 2^20) blocks raises
    InvalidArgument after the frames before it completed; it leaves no block behind
    (even with a tiny pool headroom, so its band also exhausted the mapped pool), and
    the map keeps integrating afterwards exactly like one that never saw it."""
    m = svx.ProjectionModel.spinning(256, 32, 25, 25)
    cfg = svx.MapConfig(0.1, 0.5, 2, 1 << 18)
    far = (2 ** 20) * 8 * float(np.float32(0.1)) - 3.0  # some band blocks out of range
    scans = [plane_scan(m, (0.0, 0.0, 1.2), 0.0), plane_scan(m, (far, 0.0, 1.2), 0.0),
             plane_scan(m, (0.3, 0.0, 1.2), 0.0)]
    os.environ["SVX_TEST_POOL_HEAD"] = "16"
    try:
        s = svx.VoxelStore(cfg)
    finally:
        os.environ.pop("SVX_TEST_POOL_HEAD", None)
    ref = svx.VoxelStore(cfg)
    ti, tr = svx.TsdfIntegrator(s), svx.TsdfIntegrator(ref)
    import torch
    pts = np.concatenate([p for p, _ in scans[:2]]).astype(np.float32)
    offs = np.array([0, len(scans[0][0]), len(pts)], np.uint64)
    dev = torch.from_numpy(pts).cuda()
    with pytest.raises(svx.InvalidArgument):
        s.integrate_clouds_device(m, dev.data_ptr(), offs, 3, [scans[0][1], scans[1][1]],
                                  svx.IntegratorConfig())
    tr.integrate_cloud(*scans[0], m)
    assert s.block_count() == ref.block_count()
    assert s.save_bytes() == ref.save_bytes()
    r = ti.integrate_cloud(*scans[2], m)
    r2 = tr.integrate_cloud(*scans[2], m)
    assert r.frame == 2 and r2.frame == 1
    assert (r.updated_voxels, r.new_blocks) == (r2.updated_voxels, r2.new_blocks)
    assert s.save_bytes() == ref.save_bytes()
    assert np.array_equal(s.take_dirty_blocks(0), ref.take_dirty_blocks(0))


def test_load_merges_repeated_block_records(tmp_path):
    """A snapshot that repeats a block coordinate loads as ONE block
    (VoxelStore::load calls get_or_allocate_block, voxel_store.cpp:145): the later
    TSDF wins, semantics are taken from the later record that has them; the same
    file loaded by the reference's own reader gives the same map."""
    import struct
    K = 2
    rng = np.random.default_rng(4)

    def rec(b, sem):
        t = np.zeros(512, TSDF_DTYPE)
        t["distance"] = rng.uniform(-1, 1, 512)
        t["weight"] = rng.uniform(0, 2, 512)
        out = struct.pack("<3i", *b) + t.tobytes()
        if sem is None:
            return out + b"\x00"
        return out + b"\x01" + np.full(512 * K, sem, np.float32).tobytes()

    recs = [rec((0, 0, 0), 0.25), rec((1, 0, 0), None), rec((0, 0, 0), None),
            rec((2, 0, 0), None), rec((1, 0, 0), 0.75), rec((0, 0, 0), None)]
    blob = b"SVOX1" + struct.pack("<ffIQ", 0.1, 0.5, K, len(recs)) + b"".join(recs)
    p = tmp_path / "dup.svox"
    p.write_bytes(blob)
    g = svx.VoxelStore.load(str(p), max_blocks=3)      # 3 distinct blocks fit
    assert g.block_count() == 3
    from oracle.bindings import RefMap, ref_available
    if ref_available():
        r = RefMap.load(str(p), svx.MapConfig(0.1, 0.5, K))
        assert g.save_bytes() == r.save_bytes()
    assert g.lookup_voxel((0, 0, 0))[1][0] == np.float32(0.25)
    assert g.lookup_voxel((8, 0, 0))[1][0] == np.float32(0.75)


def test_kernel_launch_counter_moves():
    s = svx.VoxelStore(svx.MapConfig(0.1, 0.5))
    m = svx.ProjectionModel.spinning(256, 32, 25, 25)
    pts, pose = plane_scan(m, (0, 0, 1.5), 0.0)
    n0 = svx.kernel_launches()
    svx.TsdfIntegrator(s).integrate_cloud(pts, pose, m)
    assert svx.kernel_launches() > n0
